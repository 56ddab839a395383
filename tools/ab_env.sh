# A/B timing of environment variants (run from the repo root through gpurun): for each config in AB_CFGS and
# each variant in AB_ENVS ("NAME=VAL" or "-" for none), the device-resident bench value, per-class gated
# times and the HBM fractions; two alternating passes.  Output: gpurun_out/ab_env.txt
mkdir -p gpurun_out; rm -f gpurun_out/ab_env.txt
for pass in 1 2; do
  for cfg in ${AB_CFGS:-walker}; do
    for ev in ${AB_ENVS:--}; do
      if [ "$ev" = "-" ]; then E=""; else E="$ev"; fi
      env $E timeout 600 python bench.py --config $cfg --steps ${AB_STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 1.5 2>/dev/null \
        | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k={n: round(v['ms']*1e3,1) for n,v in d['kernels'].items()}
h={n: round(v['frac'],3) for n,v in d['roofline'].get('hbm',{}).items()}
print('$cfg', '$ev', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', h, k)" >> gpurun_out/ab_env.txt 2>&1
    done
  done
done
cat gpurun_out/ab_env.txt
