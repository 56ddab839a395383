"""Diagnosis: per-tile timeline of the weight-gradient launch of one WLK update (eager, PDL): which tiles run
before the grid-dependency wait (critic / value groups) and when, against the actor tail."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synthdata
from paper_2312_06126_b200 import spz
cfg = sys.argv[1] if len(sys.argv) > 1 else "walker"
w = synthdata.WORKLOADS[cfg]
C = 200_000
g = spz.Replay(w.obs_dim, w.act_dim, C)
g.push(**synthdata.transitions("locomotion", w.obs_dim, w.act_dim, C))
lrn = spz.Learner(g, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=w.batch, use_graph=False)
try:
    lrn.update(w.batch, 3)
except spz.SpzError as e:
    print("warm-up:", str(e)[:80])
idx = int(os.environ.get("TRACE_IDX", "1"))  # tc_gemm launches per WLK step: critic dgrad (0), wgrad (1)
for rep in range(2):
    spz.spz_diag_tc_trace(idx + 2)
    try:
        lrn.update(w.batch, 1)
    except spz.SpzError as e:
        print("update:", str(e)[:80])
    tr, tiles, cta = spz.spz_diag_tc_trace_tiles()
    cta = cta.astype(np.int64)
    spz.spz_diag_tc_trace(0)
    tr = tr.astype(np.int64)
    T = int(tr[-1, -1, -1]); tr[-1, -1, -1] = 0
    t0 = min(tr[tr > 0].min(), cta[cta > 0].min())
    ent = (cta[:, 0][cta[:, 0] > 0] - t0) / 1e3
    wt = (cta[:, 1][cta[:, 1] > 0] - t0) / 1e3
    print(f"  CTA entry: n {ent.size} min/med/max {ent.min():.2f} {np.median(ent):.2f} {ent.max():.2f} us; entries per us:",
          " ".join(str(x) for x in np.histogram(ent, bins=np.arange(0, ent.max() + 1.0, 1.0))[0]))
    if wt.size:
        print(f"  producer past the wait: n {wt.size} min/med/max {wt.min():.2f} {np.median(wt):.2f} {wt.max():.2f} us")
    rows = []
    for c in range(160):
        for i in range(8):
            if tiles[c, i] >= 0 and tr[c, i, 0] > 0:
                rows.append((tr[c, i, 0] - t0, tr[c, i, 1] - t0, tr[c, i, 3] - t0, int(tiles[c, i]), c, tr[c, i, 2] - t0))
    rows.sort()
    print(f"launch {idx}: T={T} tiles traced {len(rows)}, CTAs {len(set(r[4] for r in rows))}")
    st = np.array([r[0] for r in rows]) / 1e3
    dn = np.array([r[2] for r in rows]) / 1e3
    tid = np.array([r[3] for r in rows])
    iss = np.array([r[1] for r in rows]) / 1e3
    acc = np.array([r[5] for r in rows]) / 1e3
    npre = int(os.environ.get("NPRE", "90"))
    for lo, hi, nm in [(0, npre, f"first {npre} tiles"), (npre, 10**9, f"tiles >= {npre}")]:
        m = (tid >= lo) & (tid < hi)
        if m.any():
            print(f"  {nm:15s}: mean producer->MMA issued {np.mean(iss[m] - st[m]):6.2f} us, issued->acc seen "
                  f"{np.mean(acc[m] - iss[m]):6.2f}, epilogue {np.mean(dn[m] - acc[m]):6.2f}")
            print(f"  {nm:15s}: n {m.sum():4d} start min/med/max {st[m].min():6.2f} {np.median(st[m]):6.2f} {st[m].max():6.2f} us"
                  f" | done min/med/max {dn[m].min():6.2f} {np.median(dn[m]):6.2f} {dn[m].max():6.2f} us")
    hist = np.histogram(st, bins=np.arange(0, st.max() + 1.0, 1.0))[0]
    print("  tile starts per us:", " ".join(str(x) for x in hist))
