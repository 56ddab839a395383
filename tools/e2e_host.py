import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import synthdata
from paper_2312_06126_b200 import spz
w = synthdata.WORKLOADS["walker"]; B = w.batch
ring = spz.Replay(w.obs_dim, w.act_dim, 1_000_000)
ring.push(**synthdata.workload_transitions(w, n=1_000_000))
lrn = spz.Learner(ring, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=B)
host = synthdata.workload_transitions(w, n=B * 4, seed=7)
pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in host.items()}
sl = lambda k: slice((k % 4) * B, (k % 4 + 1) * B)
for k in range(5):
    ring.push(**{n: v[sl(k)] for n, v in pinned.items()}); lrn.update(B, 1)
torch.cuda.synchronize()
K = 300
tp = tw = tu = 0.0
t0 = time.perf_counter()
for k in range(K):
    a = time.perf_counter(); ring.push(**{n: v[sl(k)] for n, v in pinned.items()}); b = time.perf_counter()
    if k >= 2: lrn.wait()
    c = time.perf_counter(); lrn.update_async(B, 1); d = time.perf_counter()
    tp += b - a; tw += c - b; tu += d - c
lrn.wait(); lrn.wait(); torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"per step {1e6*dt/K:.1f} us: push {1e6*tp/K:.1f}, wait {1e6*tw/K:.1f}, update_async {1e6*tu/K:.1f}")
# python marshalling alone
args = {n: v[sl(0)] for n, v in pinned.items()}
t0 = time.perf_counter()
for k in range(K): _ = {n: v[sl(k)] for n, v in pinned.items()}
print(f"dict/slices {1e6*(time.perf_counter()-t0)/K:.2f} us")
