# compute-sanitizer over the tcgen05 / TMA / mbarrier kernels (run from the repo root through gpurun).
# memcheck, racecheck (shared-memory hazards) and synccheck (barrier misuse) on the GEMM unit tests (incl. the
# dynamic tile schedule) and on small whole-update runs (fused MLP forwards, loss with deferred totals, dgrad,
# fused actor backward, pre-wait weight-gradient schedule, float4 Adam; the pipelined multi-group gather; the
# non-finite halt) in both precisions.  Summaries in gpurun_out/r2/sanitize_<tool>.log.
mkdir -p gpurun_out/r2
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  {
    echo "== $tool: GEMM unit tests"
    timeout 1500 $CS --tool $tool --target-processes all --print-limit 20 \
      python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k "not 65536" 2>&1 | tail -8
    echo "== $tool: whole-update runs (ragged multitile, WLK-shaped determinism, gather operands, non-finite halt)"
    timeout 2400 $CS --tool $tool --target-processes all --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
      -k "ragged_multitile or determinism or (learner_gather_operands_bit_exact and (22 or 30000)) or (nonfinite and 2048)" 2>&1 | tail -8
  } > gpurun_out/r2/sanitize_$tool.log 2>&1
done
