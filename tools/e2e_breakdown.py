"""Diagnostics: host-side cost of the e2e loop pieces (spz_replay_push from pinned host memory,
spz_update(B, 1) with its stats read-back), walker workload."""
import sys
import time

import numpy as np
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
for _ in range(10):
    lrn.update(B, 1)
K = 100


def timeit(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        fn(k)
    torch.cuda.synchronize()
    print(f"{name:28s} {1e6 * (time.perf_counter() - t0) / K:8.1f} us/iter")


sl = lambda k: slice((k % 4) * B, (k % 4 + 1) * B)
timeit("push pinned", lambda k: ring.push(**{n: v[sl(k)] for n, v in pinned.items()}))
timeit("push pageable", lambda k: ring.push(**{n: v[sl(k)] for n, v in host.items()}))
timeit("update(B,1)", lambda k: lrn.update(B, 1))
timeit("update(B,10)/10", lambda k: lrn.update(B, 10) if k % 10 == 0 else None)
timeit("push pinned + update", lambda k: (ring.push(**{n: v[sl(k)] for n, v in pinned.items()}), lrn.update(B, 1)))
timeit("spz_replay_info", lambda k: ring.info())
x = torch.empty(B * (2 * w.obs_dim + w.act_dim + 2), pin_memory=True)
y = torch.empty_like(x, device="cuda")
timeit("torch H2D 1.7MB pinned", lambda k: y.copy_(x, non_blocking=True))
timeit("torch H2D 1.7MB + sync", lambda k: (y.copy_(x, non_blocking=True), torch.cuda.synchronize()))
xs = [x[:B * 22], x[B * 22:B * 28], x[B * 28:B * 50], x[B * 50:B * 51], x[B * 51:B * 52]]
ys = [y[:B * 22], y[B * 22:B * 28], y[B * 28:B * 50], y[B * 50:B * 51], y[B * 51:B * 52]]
timeit("torch 5x H2D + sync", lambda k: ([b.copy_(a, non_blocking=True) for a, b in zip(xs, ys)], torch.cuda.synchronize()))
big = torch.empty(64 << 20, pin_memory=True)
bigd = torch.empty_like(big, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    bigd.copy_(big, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D bandwidth (256 MB pinned): {5 * big.numel() * 4 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
