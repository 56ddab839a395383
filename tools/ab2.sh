# A/B of library variants exp/libspz_*.so x SPZ_TC_PAIR settings over configs (device-resident bench lines).
mkdir -p gpurun_out
rm -f gpurun_out/ab2.txt
for cfg in ${AB_CONFIGS:-walker humanoid}; do
  for lib in exp/libspz_*.so; do
    for pv in ${AB_PAIR:-auto 0}; do
      if [ "$pv" = "auto" ]; then unset SPZ_TC_PAIR; else export SPZ_TC_PAIR=$pv; fi
      SPZ_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 1 2>/dev/null \
        | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k={n: round(v['ms']*1e3,1) for n,v in d['kernels'].items()}
print('$cfg $lib pair=$pv', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', k)" >> gpurun_out/ab2.txt 2>&1
    done
  done
done
unset SPZ_TC_PAIR
cat gpurun_out/ab2.txt
