# final measurement pass of a round: GPU tests, bench lines of all configs + reference arm,
# ncu launch list with DRAM traffic, ncu --set full of one K3 launch.  TAG=r02f bash tools/run_final.sh
TAG=${TAG:-r02f}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > $O/${TAG}_pytest_gpu.txt; cat $O/${TAG}_pytest_gpu.txt
timeout 900 python bench.py > $O/${TAG}_bench_cfg5.json 2> $O/${TAG}_bench_cfg5.err; tail -c 600 $O/${TAG}_bench_cfg5.json
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_cfg5_reference.json 2> $O/${TAG}_bench_cfg5_reference.err; tail -c 400 $O/${TAG}_bench_cfg5_reference.json
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 5 > $O/${TAG}_bench_cfg$c.json 2> $O/${TAG}_bench_cfg$c.err; head -c 250 $O/${TAG}_bench_cfg$c.json; echo; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file $O/${TAG}_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-fp64 --no-extras --no-cpu-baseline --e2e-steps 0 > $O/${TAG}_launches_cfg5.log 2>&1; tail -2 $O/${TAG}_launches_cfg5.log | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_tcb --launch-skip 3 -c 1 -o $O/${TAG}_tcb_ncu python tools/tcb_prof.py 1200 > $O/${TAG}_tcb_ncu.log 2>&1; tail -2 $O/${TAG}_tcb_ncu.log
