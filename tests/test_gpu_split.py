"""Actor/critic model parallelism: a critic-role learner and an actor-role learner, exchanging
parameters at every step boundary (spz_split_exchange), compute the single-learner update (Jacobi order),
checked against the oracle and against the co-located learner.  One GPU: both halves on device 0."""

import numpy as np
import pytest

import synthdata
from oracle import sac as osac, td3 as otd3
from tests.test_gpu_parity import TOL, make_rings, rel
from tests.test_gpu_sharded import make_learner

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_06126_b200 import spz  # noqa: E402


@pytest.mark.parametrize("algo,precision", [("sac", "fp32"), ("sac", "bf16"), ("td3", "fp32"), ("td3", "bf16")])
def test_split_roles_match_single_and_oracle(algo, precision):
    o, m, h, L, B, C, K = 22, 6, 256, 2, 1000, 20_000, 4
    g, r = make_rings(o, m, C)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    crit = make_learner(g, p, algo, precision, h, L, B, role=spz.SPZ_ROLE_CRITIC)
    act = make_learner(g, p, algo, precision, h, L, B, role=spz.SPZ_ROLE_ACTOR)
    full = make_learner(g, p, algo, precision, h, L, B)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=algo == "sac")
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=float(full.get("log_alpha")[0]),
                           actor_targ=p["actor"] if algo == "td3" else None)
    step = osac.sac_step if algo == "sac" else otd3.td3_step
    for k in range(K):
        sc = crit.update(B, 1)
        sa = act.update(B, 1)
        spz.spz_split_exchange(crit.h, act.h)
        sf = full.update(B, 1)
        st, so, _ = step(st, r, B, synthdata.SAMPLE_SEED, cfg)
        # each half reports its own half of the statistics
        assert abs(sc["critic_loss"] - sf["critic_loss"]) <= 1e-6 * abs(sf["critic_loss"])
        assert abs(sa["actor_loss"] - sf["actor_loss"]) <= 1e-6 * max(abs(sf["actor_loss"]), 1e-6)
    tol = TOL[precision]
    for name, side in (("q1", crit), ("q2", crit), ("q1_targ", crit), ("q2_targ", crit), ("actor", act)):
        assert rel(side.get(name), full.get(name)) <= 1e-6, name
        assert rel(side.get(name), getattr(st, name)) <= tol, name
    # the received copies are current too
    assert np.array_equal(crit.get("actor"), act.get("actor"))
    assert np.array_equal(act.get("q1"), crit.get("q1"))
    if algo == "sac":
        assert abs(float(act.get("log_alpha")[0]) - st.log_alpha) <= tol * max(1.0, abs(st.log_alpha))
        assert float(crit.get("log_alpha")[0]) == float(act.get("log_alpha")[0])
    else:
        assert rel(act.get("actor_targ"), st.actor_targ) <= tol
        assert np.array_equal(crit.get("actor_targ"), act.get("actor_targ"))
    assert crit.counters()["t_actor"] == 0 and act.counters()["t_critic"] == 0
