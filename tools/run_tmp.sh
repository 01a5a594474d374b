for L in base oneacc base oneacc; do CS_LIBPATH=ab_libs/lib$L.so timeout 300 python tools/abtime.py 5 1 2>&1 | grep warm=True; done
for L in base oneacc; do CS_NO_SCALAR=1 CS_LIBPATH=ab_libs/lib$L.so timeout 300 python tools/tcb_check.py 4096 1 2>&1 | tail -1; done
