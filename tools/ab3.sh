# w2 vs w4 (tc_gemm epilogue warps per lane quarter), alternating passes, WLK and HUM; GEMM unit tests on w4.
mkdir -p gpurun_out; rm -f gpurun_out/ab3.txt
for pass in 1 2; do
  for cfg in walker humanoid; do
    for lib in exp/libspz_w2.so exp/libspz_w4.so; do
      SPZ_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-fp32 --no-configs --min-time 2 2>/dev/null \
        | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$cfg $lib', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step')" >> gpurun_out/ab3.txt 2>&1
    done
  done
done
SPZ_LIB_PATH=$PWD/exp/libspz_w4.so timeout 600 python -m pytest tests/test_gpu_gemm.py -q 2>&1 | tail -5 >> gpurun_out/ab3.txt
cat gpurun_out/ab3.txt
