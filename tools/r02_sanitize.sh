# compute-sanitizer over the tcgen05 / TMA / mbarrier kernels (run from the repo root through gpurun).
# memcheck, racecheck (shared-memory hazards) and synccheck (barrier misuse) on the GEMM unit tests and on
# a small whole-update parity run (fused MLP forwards, loss, dgrad, fused actor backward, wgrad, Adam) in
# both precisions.  Summaries in gpurun_out/r2/sanitize_<tool>.log.
mkdir -p gpurun_out/r2
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  {
    echo "== $tool: GEMM unit tests"
    timeout 1500 $CS --tool $tool --target-processes all --print-limit 20 \
      python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "not 65536" 2>&1 | tail -8
    echo "== $tool: whole-update parity (ragged multitile, gather operands)"
    timeout 1500 $CS --tool $tool --target-processes all --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
      -k "ragged_multitile or (learner_gather_operands_bit_exact and 22)" 2>&1 | tail -8
  } > gpurun_out/r2/sanitize_$tool.log 2>&1
done
