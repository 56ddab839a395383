"""Where the Adam kernel's in-graph cost goes: per-update time of the WLK step with the full plan, with the Adam
kernel doing statistics + counters only (SPZ_DIAG_ADAM_NOWORK), and without the Adam kernel at all."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

ring = spz.Replay(22, 6, 1_000_000)
ring.push(**synthdata.transitions("locomotion", 22, 6, 1_000_000))
for label, env in (("full", {}), ("adam no element work", {"SPZ_DIAG_ADAM_NOWORK": "1"}),
                   ("no adam kernel", {"SPZ_DIAG_SKIP_OPS": "adam_polyak"})):
    for k in ("SPZ_DIAG_ADAM_NOWORK", "SPZ_DIAG_SKIP_OPS"):
        os.environ.pop(k, None)
    os.environ.update(env)
    lrn = spz.Learner(ring, precision="bf16", hidden=256, n_hidden=2, max_batch=8192)
    try:
        lrn.update(8192, 20)
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            lrn.update(8192, 300)
            best = min(best, (time.perf_counter() - t) / 300 * 1e6)
        print(f"{label:24s} {best:.1f} us/update")
    except spz.SpzError as e:
        print(label, "error", e)
    lrn.close()
