"""Diagnosis: per-(unit, layer) timelines of the fused MLP forward launches of one WLK update (eager)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

w = synthdata.WORKLOADS["walker"]
C = 200_000
g = spz.Replay(w.obs_dim, w.act_dim, C)
g.push(**synthdata.transitions("locomotion", w.obs_dim, w.act_dim, C))
lrn = spz.Learner(g, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=w.batch, use_graph=False)
lrn.update(w.batch, 3)
for k, nm in enumerate(["actor_fwd_mlp", "critic_fwd_mlp"]):
    spz.spz_diag_mlp_trace(k + 2)
    lrn.update(w.batch, 1)
    tr = spz.spz_diag_mlp_trace(0, read=True).astype(np.int64)  # [cta, unit, layer, event]
    if (tr > 0).sum() == 0:
        print(nm, "no trace")
        continue
    t0 = tr[tr > 0].min()
    nl = int((tr[:, 0, :, 0] > 0).any(axis=0).sum())
    print(f"{nm}: span {(tr.max() - t0) / 1e3:.2f} us, layers {nl}")
    for l in range(nl):
        ok = (tr[:, :, l, 0] > 0) & (tr[:, :, l, 3] > 0)
        if not ok.any():
            continue
        s, i, a, d, f0, f1 = (tr[:, :, l, e][ok] for e in range(6))
        print(f"  layer {l}: MMA issue {(i - s).mean() / 1e3:5.2f} us (first slab {(f0 - s).mean() / 1e3:5.2f}, last slab "
              f"{(f1 - s).mean() / 1e3:5.2f}) | acc latency after issue {(a - i).mean() / 1e3:5.2f} | "
              f"epilogue {(d - a).mean() / 1e3:5.2f} | start (from t0) {(s - t0).mean() / 1e3:6.2f}")
    for l in range(1, nl):
        ok = (tr[:, :, l, 0] > 0) & (tr[:, :, l - 1, 3] > 0)
        gap = (tr[:, :, l, 0] - tr[:, :, l - 1, 3])[ok]
        print(f"  handoff layer {l - 1} epilogue done -> layer {l} MMA start: {gap.mean() / 1e3:5.2f} us")
    units = (tr[:, :, 0, 0] > 0).sum(axis=1)
    first = tr[:, 0, 0, 0][tr[:, 0, 0, 0] > 0]
    print(f"  units/CTA max {units.max()}, first MMA start spread {(first.max() - first.min()) / 1e3:.2f} us")
    for u in range(int(units.max())):
        ok = tr[:, u, 0, 0] > 0
        st = (tr[:, u, 0, 0][ok] - t0).mean() / 1e3
        en = (tr[:, u, nl - 1, 3][ok & (tr[:, u, nl - 1, 3] > 0)] - t0).mean() / 1e3
        print(f"  unit {u}: mean start {st:6.2f} us, mean end {en:6.2f} us")

# CTA 0's event sequence of the last traced launch (the critic forward): unit, layer, event, us from t0
names = {0: "mma_start", 4: "mma_first_kb", 5: "mma_last_kb", 1: "mma_issued", 2: "epi_start", 3: "epi_done"}
for cta in (0, 1, 100):
    ev = [(int(tr[cta, u, l, e]), u, l, names[e]) for u in range(tr.shape[1]) for l in range(tr.shape[2])
          for e in range(tr.shape[3]) if tr[cta, u, l, e] > 0]
    ev.sort()
    print(f"CTA {cta}:", "; ".join(f"u{u}L{l} {n} {(t - t0) / 1e3:.2f}" for t, u, l, n in ev))
