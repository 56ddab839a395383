# CTA-pair GEMM on / off (SPZ_TC_PAIR=0) at the wide configs, device-resident bench lines; then HUM / TD3 parity.
mkdir -p gpurun_out
rm -f gpurun_out/pair_ab.txt
for cfg in humanoid humanoid_td3; do
  for pv in 0 auto; do
    if [ "$pv" = "0" ]; then export SPZ_TC_PAIR=0; else unset SPZ_TC_PAIR; fi
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 1 2>/dev/null \
      | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k={n: round(v['ms']*1e3,1) for n,v in d['kernels'].items()}
print('$cfg pair=$pv', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), k)" >> gpurun_out/pair_ab.txt 2>&1
  done
done
unset SPZ_TC_PAIR
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "humanoid_full_size or td3_full_size or walker_full_size" 2>&1 | tail -5 >> gpurun_out/pair_ab.txt
cat gpurun_out/pair_ab.txt
