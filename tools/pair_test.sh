timeout 240 python -m pytest tests/test_gpu_gemm.py -q -x -k "cta_pair" 2>&1 | tail -15 > gpurun_out/pair1.txt
echo "rc=$?" >> gpurun_out/pair1.txt
nvidia-smi --query-gpu=name,utilization.gpu --format=csv >> gpurun_out/pair1.txt
