# same-box A/B of the warm-start GEMM builds (tools/warm_gemm_ab.py)
timeout 180 python tools/warm_gemm_ab.py 32768 2>&1 | tail -3
for L in spa2; do CS_LIBPATH=ab_libs/lib$L.so timeout 180 python tools/warm_gemm_ab.py 32768 2>&1 | tail -3; done
timeout 300 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "warm" 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:warm_gemm_tc --launch-skip 3 -c 1 -o gpurun_out/r02e_wg_ncu2 python tools/warm_gemm_ab.py 8192 > gpurun_out/r02e_wg_ncu2.log 2>&1
