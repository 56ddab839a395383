"""Marginal cost of each op class inside the CUDA-graph replay of the WLK SAC update.

For each class, a learner is built with SPZ_DIAG_SKIP_OPS=<class> (diagnostics: that op is dropped,
results are wrong) and the per-update time is compared with the full plan.  Prints one line per class.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

CLASSES = ["gather", "actor_fwd_mlp", "critic_fwd_mlp", "critic_loss", "critic_dgrad_gemm",
           "actor_bwd_fused", "wgrad_gemm", "adam_polyak"]


def per_update_ms(ring, skip, B=8192, K=300, reps=3):
    if skip:
        os.environ["SPZ_DIAG_SKIP_OPS"] = skip
    else:
        os.environ.pop("SPZ_DIAG_SKIP_OPS", None)
    lrn = spz.Learner(ring, precision="bf16", hidden=256, n_hidden=2, max_batch=B)
    try:
        lrn.update(B, 20)
    except spz.SpzError:  # e.g. without critic_loss Adam has no bias-correction snapshot
        return float("nan")
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        try:
            lrn.update(B, K)
        except spz.SpzError as e:
            return float("nan")
        best = min(best, (time.perf_counter() - t) / K * 1e3)
    return best


def main():
    o, m = 22, 6
    ring = spz.Replay(o, m, 1_000_000)
    ring.push(**synthdata.transitions("locomotion", o, m, 1_000_000))
    full = per_update_ms(ring, None)
    print(f"full plan: {full * 1e3:.1f} us/update")
    for c in CLASSES:
        t = per_update_ms(ring, c)
        print(f"  without {c:26s} {t * 1e3:7.1f} us  -> marginal {1e3 * (full - t):6.1f} us")


if __name__ == "__main__":
    main()
