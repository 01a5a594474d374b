# same-box A/B of the in-tree library ("default") against ab_libs/libbase.so (tools/ab_build.sh),
# bitwise check first, then the per-phase split of ab_libs/libclk.so when present
timeout 600 python tools/bitwise_ab.py ab_libs/libbase.so default ${1:-4096} 2>&1 | tail -4
for L in base default base default; do
  if [ $L = default ]; then timeout 300 python tools/abtime.py 5 2 2>&1 | grep warm=True
  else CS_LIBPATH=ab_libs/lib$L.so timeout 300 python tools/abtime.py 5 2 2>&1 | grep warm=True; fi
done
if [ -f ab_libs/libclk.so ]; then CS_LIBPATH=ab_libs/libclk.so timeout 300 python tools/tcb_split.py 4096 1 2>&1 | tail -18; fi
