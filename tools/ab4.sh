mkdir -p gpurun_out; rm -f gpurun_out/ab4.txt
for pass in 1 2; do
  for cfg in walker humanoid ant; do
    for lib in exp/libspz_w2.so exp/libspz_wauto.so; do
      SPZ_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 2 2>/dev/null \
        | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg $lib', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step')" >> gpurun_out/ab4.txt 2>&1
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x -k "gemm or walker_full or ragged or pendulum or td3_parity or pair_schedule or humanoid_shape" 2>&1 | tail -4 >> gpurun_out/ab4.txt
cat gpurun_out/ab4.txt
