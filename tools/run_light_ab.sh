set -x
for L in base light14 light12 base light14 light12; do CS_LIBPATH=ab_libs/lib$L.so timeout 300 python tools/abtime.py 5 2 2>&1 | grep warm=True; done
for L in base light14 light12; do CS_NO_SCALAR=1 CS_LIBPATH=ab_libs/lib$L.so timeout 300 python tools/tcb_check.py 2048 1 2>&1 | tail -1; done
CS_LIBPATH=ab_libs/libclk14.so timeout 300 python tools/tcb_split.py 4096 1 2>&1 | tail -25
