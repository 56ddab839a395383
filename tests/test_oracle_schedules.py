"""Schedule equivalence in fp64: sharded == split == single."""

import numpy as np
import pytest

from oracle import sac, schedules, td3
from tests.test_oracle_sac import small_problem


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _assert_same(a, b, tol=1e-12):
    for k in ("actor", "q1", "q2", "q1_targ", "q2_targ"):
        assert _rel(getattr(a, k), getattr(b, k)) <= tol, k
    if a.actor_targ is not None:
        assert _rel(a.actor_targ, b.actor_targ) <= tol
    assert abs(a.log_alpha - b.log_alpha) <= tol * max(1.0, abs(b.log_alpha))
    for k in a.opt:
        assert _rel(a.opt[k].m, b.opt[k].m) <= tol or np.linalg.norm(b.opt[k].m) == 0
        assert a.opt[k].t == b.opt[k].t


@pytest.mark.parametrize("algo", ["sac", "td3"])
@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_sharded_equals_single(algo, G):
    cfg, r, st = small_problem(algo)
    step = sac.sac_step if algo == "sac" else td3.td3_step
    a, b = st.copy(), st.copy()
    B = 37
    for _ in range(3):
        a, sa, ia = step(a, r, B, 6126, cfg)
        b, sb, ib = schedules.sharded_step(b, r, B, 6126, cfg, G, algo=algo)
        assert np.array_equal(ia, ib)
        for k in sa:
            assert abs(sa[k] - sb[k]) <= 1e-12 * max(1.0, abs(sa[k]))
    _assert_same(b, a)


@pytest.mark.parametrize("algo", ["sac", "td3"])
def test_split_equals_single(algo):
    cfg, r, st = small_problem(algo)
    step = sac.sac_step if algo == "sac" else td3.td3_step
    a, b = st.copy(), st.copy()
    for _ in range(4):
        a, sa, _ = step(a, r, 32, 6126, cfg)
        b, sb, _ = schedules.split_step(b, r, 32, 6126, cfg, algo=algo)
        for k in sa:
            assert abs(sa[k] - sb[k]) <= 1e-12 * max(1.0, abs(sa[k]))
    _assert_same(b, a, tol=0.0)
