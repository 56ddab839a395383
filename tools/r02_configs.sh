# Bench lines of every BASELINE config on one B200 (run from the repo root through gpurun): default precision bf16
# (+ the fp32 key), parity + cpu_baseline beside each.  Outputs gpurun_out/r2/bench_<config>.json
mkdir -p gpurun_out/r2
for c in pendulum walker ant humanoid humanoid_td3; do
  timeout 1500 python bench.py --config $c > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
done
ls -la gpurun_out/r2/bench_*
