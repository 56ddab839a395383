# Round-end capture on one B200 (run from the repo root through gpurun): GPU tests, default bench, f4 bench lines,
# ncu launch lists and one ncu --set full capture of the fused MLP forward.  Outputs land in gpurun_out/.
mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log > gpurun_out/r01_bench_final.json
timeout 300 python bench.py --algo sacv1 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01_bench_sacv1.json
timeout 300 python bench.py --algo ddpg --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01_bench_ddpg.json
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -s 90 -c 40 --csv --log-file gpurun_out/r01_launches_warm_final.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 90 -c 40 --csv --log-file gpurun_out/r01_launches_basic.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_mlp -s 20 -c 2 -o gpurun_out/mlp_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/
