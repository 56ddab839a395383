"""Per-update time of the WLK SAC update (CUDA-graph replay, host-timed over K updates, best of 3) under each
environment setting given on the command line ("NAME=VAL" or "-"); diagnostics settings may make the results
wrong -- only the time is reported."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402


def per_update_us(ring, w, K=300, reps=3):
    lrn = spz.Learner(ring, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=w.batch)
    try:
        lrn.update(w.batch, 20)
        best = 1e9
        for _ in range(reps):
            t = time.perf_counter()
            lrn.update(w.batch, K)
            best = min(best, (time.perf_counter() - t) / K * 1e6)
        return best, ""
    except spz.SpzError as e:
        return float("nan"), str(e)[:120]


def main():
    cfg = os.environ.get("CFG", "walker")
    w = synthdata.WORKLOADS[cfg]
    C = 1_000_000
    ring = spz.Replay(w.obs_dim, w.act_dim, C)
    ring.push(**synthdata.transitions("locomotion", w.obs_dim, w.act_dim, C))
    for rep in range(2):
        for ev in sys.argv[1:]:
            saved = dict(os.environ)
            if ev != "-":
                k, v = ev.split("=", 1)
                os.environ[k] = v
            t, err = per_update_us(ring, w)
            os.environ.clear()
            os.environ.update(saved)
            print(f"{cfg} {ev:28s} {t:7.1f} us/update {err}", flush=True)


if __name__ == "__main__":
    main()
