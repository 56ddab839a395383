mkdir -p gpurun_out; rm -f gpurun_out/ab5.txt
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_policy.py tests/test_gpu_sharded.py tests/test_gpu_split.py -q 2>&1 | tail -4 >> gpurun_out/ab5.txt
cat gpurun_out/ab5.txt
