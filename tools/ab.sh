# A/B timing of library variants exp/libspz_*.so (run from the repo root through gpurun): the default WLK
# bench (device-resident value + gated per-class times), two alternating passes.  Output: gpurun_out/ab.txt
mkdir -p gpurun_out
CFG=${AB_ARGS:-""}
for pass in 1 2; do
  for lib in exp/libspz_*.so; do
    SPZ_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-fp32 --min-time 1 $CFG 2>/dev/null \
      | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k={n: round(v['ms']*1e3,1) for n,v in d['kernels'].items()}
print('$lib', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', k)" >> gpurun_out/ab.txt 2>&1
  done
done
cat gpurun_out/ab.txt
