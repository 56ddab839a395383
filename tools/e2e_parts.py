"""Diagnostics: where the end-to-end loop's time goes at WLK (host-timed, 300 steps): the bench's e2e loop
(push_async + wait + update_async, two updates in flight), the same with three in flight, pushes alone,
asynchronous updates alone, and the device-resident graph replay."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

w = synthdata.WORKLOADS["walker"]
B = w.batch
ring = spz.Replay(w.obs_dim, w.act_dim, 1_000_000)
ring.push(**synthdata.workload_transitions(w, n=1_000_000))
lrn = spz.Learner(ring, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=B)
host = synthdata.workload_transitions(w, n=B * 4, seed=7)
pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in host.items()}
sl = lambda k: slice((k % 4) * B, (k % 4 + 1) * B)
for k in range(5):
    ring.push(**{n: v[sl(k)] for n, v in pinned.items()})
    lrn.update(B, 1)
K = 300


def run(name, step, tail=lambda: None):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(K):
            step(k)
        tail()
        ring.sync()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / K * 1e6)
    print(f"{name:44s} {best:7.1f} us/step  ({B / best:.1f}M frames/s)", flush=True)


def e2e(inflight):
    def step(k):
        ring.push(**{n: v[sl(k)] for n, v in pinned.items()}, wait=False)
        if k >= inflight:
            lrn.wait()
        lrn.update_async(B, 1)

    def tail():
        for _ in range(min(inflight, K)):
            lrn.wait()
    return step, tail


run("e2e, 2 in flight (bench)", *e2e(2))
run("pushes only (push_async)", lambda k: ring.push(**{n: v[sl(k)] for n, v in pinned.items()}, wait=False))
upd_step, upd_tail = (lambda k: (lrn.wait() if k >= 2 else None, lrn.update_async(B, 1))), (lambda: (lrn.wait(), lrn.wait()))
run("updates only (update_async, 2 in flight)", upd_step, upd_tail)
run("device-resident spz_update(B, 300) / 300", lambda k: lrn.update(B, K) if k == 0 else None)
