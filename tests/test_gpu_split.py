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


def _split_worker(rank, world, port, q, B, K, algo):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_06126_b200.dist import broadcast_bytes
    uid = broadcast_bytes(spz.spz_nccl_unique_id() if rank == 0 else None)
    o, m, h, L, C = 22, 6, 256, 2, 50_000
    tr = synthdata.transitions("locomotion", o, m, C)
    g = spz.Replay(o, m, C, device=rank)
    g.push(**tr)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    role = spz.SPZ_ROLE_CRITIC if rank < world // 2 else spz.SPZ_ROLE_ACTOR
    lrn = make_learner(g, p, algo, "bf16", h, L, B, device=rank, world_size=world, rank=rank, role=role,
                       n_critic_ranks=world // 2, n_actor_ranks=world - world // 2, nccl_unique_id=uid)
    lrn.update(B, K)
    q.put((rank, lrn.get("actor"), lrn.get("q1")))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL split test needs >= 2 GPUs")
@pytest.mark.parametrize("algo", ["sac", "td3"])
def test_nccl_split_roles_match_single_gpu(algo):
    """Critic group and actor group on different GPUs (in-graph NCCL exchange) == one co-located learner."""
    import os
    import torch.multiprocessing as mp
    world = 4 if torch.cuda.device_count() >= 4 else 2
    B, K = 4096, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    ps = [ctx.Process(target=_split_worker, args=(r, world, port, q, B, K, algo)) for r in range(world)]
    for pr in ps:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in ps], key=lambda x: x[0])
    for pr in ps:
        pr.join(timeout=60)
    for r in range(1, world):  # every rank holds identical (exchanged) parameters
        assert np.array_equal(res[r][1], res[0][1]) and np.array_equal(res[r][2], res[0][2])
    o, m, h, L, C = 22, 6, 256, 2, 50_000
    g, _ = make_rings(o, m, C)
    single = make_learner(g, synthdata.init_params(o, m, h, L, algo=algo), algo, "bf16", h, L, B)
    single.update(B, K)
    assert rel(res[0][1], single.get("actor")) < 2e-2 and rel(res[0][2], single.get("q1")) < 2e-2
