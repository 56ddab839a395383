"""Per-tile timelines (producer start, MMA done, epilogue start, epilogue done) of every tcgen05 GEMM launch of one
eager HUM update (3x512, B 65536): is a launch mainloop- or epilogue-bound?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

w = synthdata.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "humanoid"]
g = spz.Replay(w.obs_dim, w.act_dim, 300_000)
g.push(**synthdata.transitions("locomotion", w.obs_dim, w.act_dim, 300_000))
lrn = spz.Learner(g, algo=w.algo, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=w.batch, use_graph=False)
lrn.update(w.batch, 2)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 14):
    spz.spz_diag_tc_trace(2 + i)
    lrn.update(w.batch, 1)
    tr = spz.spz_diag_tc_trace(0, read=True).astype(np.int64)
    if (tr > 0).sum() == 0:
        print(f"launch {i}: no trace")
        continue
    t0 = tr[tr > 0].min()
    prod, mma, acc, done = (tr[:, :, e] for e in range(4))
    ok = (prod > 0) & (done > 0)
    n = ok.sum(axis=1)
    # tile i+1's mainloop runs while tile i's epilogue drains: bound = max(mainloop, epilogue) per tile
    print(f"launch {i}: tiles traced {ok.sum()} (<= 8 per CTA), mainloop {((mma - prod)[ok]).mean() / 1e3:.2f} us, "
          f"acc wait {((acc - mma)[ok]).mean() / 1e3:.2f} us, epilogue {((done - acc)[ok]).mean() / 1e3:.2f} us, "
          f"tile period {np.diff(np.where(ok, done, np.nan), axis=1)[:, :].__array__()[~np.isnan(np.diff(np.where(ok, done, np.nan), axis=1))].mean() / 1e3 if (n > 1).any() else float('nan'):.2f} us, "
          f"span {(done[ok].max() - t0) / 1e3:.1f} us")
