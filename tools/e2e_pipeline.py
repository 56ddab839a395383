"""Diagnostics: per-step cost of the e2e loop (push + update_async / wait, two updates in flight) with
push sizes 0, 1 and B rows from pinned memory, WLK shapes."""
import sys
import time

import torch

sys.path.insert(0, ".")
import synthdata
from paper_2312_06126_b200 import spz

w = synthdata.WORKLOADS["walker"]
B = w.batch
ring = spz.Replay(w.obs_dim, w.act_dim, 200_000)
ring.push(**synthdata.workload_transitions(w, n=200_000))
lrn = spz.Learner(ring, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=B)
host = synthdata.workload_transitions(w, n=B * 4, seed=7)
pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in host.items()}
lrn.update(B, 10)
K = 200
for n in (0, 1, 1024, B):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        if n:
            o = (k % 4) * B
            ring.push(**{a: v[o:o + n] for a, v in pinned.items()})
        if k >= 2:
            lrn.wait()
        lrn.update_async(B, 1)
    lrn.wait()
    lrn.wait()
    torch.cuda.synchronize()
    print(f"push {n:5d} rows: {1e6 * (time.perf_counter() - t0) / K:7.1f} us/step")
