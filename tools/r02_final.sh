# Round-2 end capture on one B200 (run from the repo root through gpurun): GPU tests, smoke, default bench,
# the batch-size sweep, the ncu launch list and one ncu --set full capture of a WLK update.
mkdir -p gpurun_out/r2f
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r2f/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err
timeout 900 python bench.py --sweep --no-cpu-baseline --no-e2e --no-fp32 --no-configs > gpurun_out/r2f/sweep.json 2> /dev/null
bash tools/r02_capture.sh > gpurun_out/r2f/cap.log 2>&1
mv gpurun_out/r2/launches.csv gpurun_out/r2f/ 2>/dev/null; mv gpurun_out/r2/full.ncu-rep gpurun_out/r2f/ 2>/dev/null
ls -la gpurun_out/r2f
