"""Batch-size adaptation: spz_tune_batch probes an
ascending ladder, reports frames/s = B x updates/s, stops past the peak, and with restore leaves the
learner exactly as it was."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402


def learner(C=40_000, max_batch=16384):
    g = spz.Replay(22, 6, C)
    g.push(**synthdata.transitions("locomotion", 22, 6, C))
    return g, spz.Learner(g, precision="bf16", hidden=256, n_hidden=2, max_batch=max_batch)


def test_tune_points_and_choice():
    g, lrn = learner()
    ladder = [256, 1024, 4096, 8192, 16384]
    best, pts = lrn.tune_batch(ladder, warmup=2, steps=10, tol=1.0)  # tol 1: never stops early
    assert [p["batch"] for p in pts] == ladder
    for p in pts:
        assert p["updates_per_s"] > 0 and abs(p["frames_per_s"] - p["batch"] * p["updates_per_s"]) <= 1e-9 * p["frames_per_s"]
        assert abs(p["ms_per_update"] * p["updates_per_s"] - 1e3) < 1e-6
    assert best == max(pts, key=lambda p: p["frames_per_s"])["batch"]
    # at small batches the fixed per-update cost dominates, so frames/s grows with B
    assert pts[-1]["frames_per_s"] > pts[0]["frames_per_s"]
    # an update-frequency floor excludes the batches that cannot meet it
    hz = sorted(p["updates_per_s"] for p in pts)[len(pts) // 2]
    best2, pts2 = lrn.tune_batch(ladder, warmup=2, steps=10, tol=1.0, min_update_hz=hz)
    ok = [p for p in pts2 if p["updates_per_s"] >= hz]
    assert best2 == max(ok, key=lambda p: p["frames_per_s"])["batch"]


def test_tune_restore_is_exact():
    g, a = learner()
    _, b = learner()
    a.tune_batch([512, 2048, 8192], warmup=1, steps=3, tol=1.0, restore=True)
    assert a.counters()["step"] == 0
    sa, sb = a.update(2048, 4), b.update(2048, 4)
    assert sa == sb
    for n in ("actor", "q1", "q2", "q1_targ"):
        assert np.array_equal(a.get(n), b.get(n))


def test_tune_errors():
    g, lrn = learner(C=3000, max_batch=4096)
    with pytest.raises(spz.SpzError) as e:
        lrn.tune_batch([1024, 512])
    assert e.value.status == spz.SPZ_EINVAL
    with pytest.raises(spz.SpzError) as e:
        lrn.tune_batch([1024, 4000], warmup=1, steps=1)  # fill 3000 < 4000
    assert e.value.status == spz.SPZ_ENODATA
