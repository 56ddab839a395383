"""Diagnosis: per-tile timelines of every tcgen05 GEMM launch of one WLK update (eager)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synthdata
from paper_2312_06126_b200 import spz
w = synthdata.WORKLOADS["walker"]
C = 200_000
g = spz.Replay(w.obs_dim, w.act_dim, C)
g.push(**synthdata.transitions("locomotion", w.obs_dim, w.act_dim, C))
lrn = spz.Learner(g, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=w.batch, use_graph=False)
lrn.update(w.batch, 3)
names = ["actor_fwd0", "actor_fwd1", "actor_head", "critic_fwd0", "critic_fwd1", "critic_dgrad", "input_dgrad",
         "actor_dgrad_head", "actor_dgrad1", "wgrad"]
for k, nm in enumerate(names):
    spz.spz_diag_tc_trace(k + 2)
    lrn.update(w.batch, 1)
    tr = spz.spz_diag_tc_trace(0, read=True).astype(np.int64)
    T = int(tr[-1, -1, -1]); tr[-1, -1, -1] = 0
    if (tr > 0).sum() == 0:
        print(nm, "no trace"); continue
    t0 = tr[tr > 0].min()
    prod, mma, acc, done = [tr[:, :, i] for i in range(4)]
    ok = (prod > 0) & (mma > 0)
    okd = ok & (done > 0)
    ntiles = ok.sum(axis=1)
    epi = ((done - acc)[okd]).mean() / 1e3 if okd.any() else float("nan")
    last = (done[okd].max() if okd.any() else mma[ok].max()) - t0
    print(f"{nm:16s} T={T:4d} tiles/cta max {ntiles.max()} | first mainloop {(mma[:,0]-prod[:,0])[ok[:,0]].mean()/1e3:5.2f} us | "
          f"mean mainloop {((mma-prod)[ok]).mean()/1e3:5.2f} | mean epi {epi:5.2f} | span {last/1e3:6.2f} us")
