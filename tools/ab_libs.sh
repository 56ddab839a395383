timeout 120 python tools/write_bw.py
for lib in base ch16 new; do
  for cfg in walker humanoid_td3 humanoid; do
    SPZ_LIB_PATH=$PWD/exp/libspz_$lib.so timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 1.5 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k={n: round(v['ms']*1e3,1) for n,v in d['kernels'].items() if n in ('gather','adam_polyak')}
h={n: round(v['frac'],3) for n,v in d['roofline'].get('hbm',{}).items()}
print('$lib $cfg', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', h, k)"
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "nonfinite or gather or generated or full_size or mutation or td3_parity or ddpg" 2>&1 | tail -3
