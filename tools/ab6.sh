# A/B of library variants exp/libspz_*.so over configs, AB_PASSES alternating passes (device-resident bench
# lines, default SPZ_TC_PAIR).  Output: gpurun_out/ab6.txt
mkdir -p gpurun_out
rm -f gpurun_out/ab6.txt
for pass in $(seq ${AB_PASSES:-2}); do
  for cfg in ${AB_CONFIGS:-walker humanoid}; do
    for lib in exp/libspz_*.so; do
      SPZ_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $cfg --steps ${AB_STEPS:-50} --warmup 10 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 1 2>/dev/null \
        | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k={n: round(v['ms']*1e3,1) for n,v in d['kernels'].items()}
print('$cfg $lib', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', k)" >> gpurun_out/ab6.txt 2>&1
    done
  done
done
cat gpurun_out/ab6.txt
