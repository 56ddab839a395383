# Round-2 profile capture on one B200 (run from the repo root through gpurun).  Outputs in gpurun_out/r2/:
#   launches.csv  -- ncu launch list (gpu__time_duration per launch, clocks free) of the bench command
#   full.ncu-rep  -- ncu --set full of one launch of each kernel class of a WLK update (cold L2, serialised)
mkdir -p gpurun_out/r2
B="python bench.py --steps 5 --warmup 3 --reps 1 --min-time 0 --no-cpu-baseline --no-e2e --no-fp32"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -s 60 -c 48 --csv --log-file gpurun_out/r2/launches.csv $B > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -s 60 -c 8 -o gpurun_out/r2/full $B > /dev/null 2>&1
ls -la gpurun_out/r2/
