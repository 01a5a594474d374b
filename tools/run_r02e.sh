set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r02e_pytest.log
cat gpurun_out/r02e_pytest.log
timeout 600 python bench.py > gpurun_out/r02e_bench_cfg5.json 2> gpurun_out/r02e_bench_cfg5.err
tail -c 3000 gpurun_out/r02e_bench_cfg5.json
timeout 200 python tools/warm_gemm_ab.py 32768 2>&1 | tail -3 > gpurun_out/r02e_warm_gemm_ab.txt
cat gpurun_out/r02e_warm_gemm_ab.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:warm_gemm_tc --launch-skip 3 -c 1 -o gpurun_out/r02e_wg_ncu python tools/warm_gemm_ab.py 8192 > gpurun_out/r02e_wg_ncu.log 2>&1
tail -3 gpurun_out/r02e_wg_ncu.log
