"""Cost of one kernel boundary inside the graph replay: the WLK update with k extra empty PDL kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

o, m, B = 22, 6, 8192
ring = spz.Replay(o, m, 1_000_000)
ring.push(**synthdata.transitions("locomotion", o, m, 1_000_000))
base = None
for k in (0, 4, 16):
    os.environ["SPZ_DIAG_NOOP_OPS"] = str(k)
    lrn = spz.Learner(ring, precision="bf16", hidden=256, n_hidden=2, max_batch=B)
    lrn.update(B, 20)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        lrn.update(B, 300)
        best = min(best, (time.perf_counter() - t) / 300 * 1e6)
    base = best if base is None else base
    print(f"{k:3d} extra empty kernels: {best:7.1f} us/update  (+{(best - base) / max(k, 1):.2f} us per boundary)")
