"""Cost of one kernel boundary inside the graph-replayed WLK update: SPZ_DIAG_NOOP_OPS=k appends k empty PDL
kernels (148 x 128 threads) to every step; per-update time against k."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

ring = spz.Replay(22, 6, 1_000_000)
ring.push(**synthdata.transitions("locomotion", 22, 6, 1_000_000))
for k in (0, 1, 2, 4, 8):
    if k:
        os.environ["SPZ_DIAG_NOOP_OPS"] = str(k)
    else:
        os.environ.pop("SPZ_DIAG_NOOP_OPS", None)
    lrn = spz.Learner(ring, precision="bf16", hidden=256, n_hidden=2, max_batch=8192)
    lrn.update(8192, 20)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        lrn.update(8192, 300)
        best = min(best, (time.perf_counter() - t) / 300 * 1e6)
    print(f"noop kernels per step {k}: {best:.1f} us/update")
    lrn.close()
