"""Row-sharded (data-parallel) update: the W ranks' local gradients and loss totals add up to the
full-batch ones (oracle), and -- with >= 2 GPUs -- the NCCL group equals the single-GPU learner."""

import os

import numpy as np
import pytest

import synthdata
from oracle import mlp, sac as osac, td3 as otd3
from tests.test_gpu_parity import make_rings, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_06126_b200 import spz  # noqa: E402


def gred_layout(grads, cfg, algo):
    """Oracle gradients in the learner's contiguous gradient-buffer order (q1, q2, actor; W then b per layer,
    each tensor padded to 16 floats)."""
    out = []
    shapes = {"q1": osac.critic_shapes(cfg), "q2": osac.critic_shapes(cfg), "actor": osac.actor_shapes(cfg, td3=algo == "td3")}
    for name in ("q1", "q2", "actor"):
        if name not in grads:
            continue
        for W, b in mlp.unflatten(grads[name], shapes[name]):
            for t in (W.ravel(), b):
                pad = (-t.size) % 16
                out.append(np.concatenate([t, np.zeros(pad)]))
    return np.concatenate(out)


def make_learner(g, p, algo, precision, h, L, B, **kw):
    lrn = spz.Learner(g, algo=algo, precision=precision, hidden=h, n_hidden=L, max_batch=B, **kw)
    lrn.set("actor", p["actor"])
    lrn.set("q1", p["q1"])
    lrn.set("q2", p["q2"])
    lrn.set("q1_targ", p["q1"])
    lrn.set("q2_targ", p["q2"])
    if algo == "td3":
        lrn.set("actor_targ", p["actor"])
    return lrn


@pytest.mark.parametrize("algo,precision,W", [("sac", "fp32", 2), ("sac", "bf16", 3), ("td3", "fp32", 2), ("td3", "bf16", 2),
                                              ("sac", "fp32", 5)])
def test_local_shard_gradients_sum_to_full_batch(algo, precision, W):
    o, m, h, L, B, C = 22, 6, 128, 2, 1000, 20_000
    g, r = make_rings(o, m, C)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=algo == "sac")
    # raw-gradient comparison: bf16 operand rounding is not averaged out by Adam here, so the bf16 bound is
    # the 2e-2 parameter bound widened to 5e-2 (the fp32 runs hold the 1e-4 bound)
    tol = 1e-4 if precision == "fp32" else 5e-2
    tot, stat = None, None
    for rk in range(W):
        lrn = make_learner(g, p, algo, precision, h, L, B, world_size=W, rank=rk, comm_mode=1)
        lrn.update(B, 1)
        gr = lrn.debug("Gred").astype(np.float64)
        ss = lrn.debug("statsum")[:5].copy()
        tot = gr if tot is None else tot + gr
        stat = ss if stat is None else stat + ss
        del lrn
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=np.log(0.2),
                           actor_targ=p["actor"] if algo == "td3" else None)
    idx, batch = r.sample(B, synthdata.SAMPLE_SEED, 0)
    if algo == "sac":
        eps, eps2 = osac.draw_noise(synthdata.SAMPLE_SEED, 0, B, m)
        grads, sums = osac.sac_grads(st, batch, eps, eps2, cfg, B)
    else:
        xi = otd3.draw_smoothing(synthdata.SAMPLE_SEED, 0, B, cfg)
        grads, sums = otd3.td3_grads(st, batch, xi, cfg, B, 0)
    ref = gred_layout(grads, cfg, algo)
    assert rel(tot[:ref.size], ref) <= tol, rel(tot[:ref.size], ref)
    # loss totals: sum (q1-y)^2 + (q2-y)^2, sum q1, sum q2 (+ SAC actor terms)
    assert abs(stat[0] - sums["lq"]) <= tol * abs(sums["lq"])
    assert abs(stat[1] - sums["q1"]) <= tol * max(abs(sums["q1"]), B * 1e-2)
    if algo == "sac":
        assert abs(stat[4] - sums["logp"]) <= tol * abs(sums["logp"])


def _nccl_worker(rank, world, port, q, B, K):
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
    p = synthdata.init_params(o, m, h, L)
    lrn = make_learner(g, p, "sac", "bf16", h, L, B, device=rank, world_size=world, rank=rank, nccl_unique_id=uid)
    s = lrn.update(B, K)
    q.put((rank, s, lrn.get("actor"), lrn.get("q1")))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL group test needs >= 2 GPUs")
def test_nccl_group_matches_single_gpu():
    import torch.multiprocessing as mp
    B, K, world = 4096, 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    ps = [ctx.Process(target=_nccl_worker, args=(r, world, port, q, B, K)) for r in range(world)]
    for pr in ps:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in ps], key=lambda x: x[0])
    for pr in ps:
        pr.join(timeout=60)
    # identical parameters on every rank
    assert np.array_equal(res[0][2], res[1][2]) and np.array_equal(res[0][3], res[1][3])
    o, m, h, L, C = 22, 6, 256, 2, 50_000
    g, _ = make_rings(o, m, C)
    single = make_learner(g, synthdata.init_params(o, m, h, L), "sac", "bf16", h, L, B)
    s1 = single.update(B, K)
    assert rel(res[0][2], single.get("actor")) < 2e-2 and rel(res[0][3], single.get("q1")) < 2e-2
    assert abs(res[0][1]["critic_loss"] - s1["critic_loss"]) < 2e-2 * abs(s1["critic_loss"])


@pytest.mark.parametrize("algo,precision", [("sac", "bf16"), ("td3", "fp32")])
def test_single_rank_nccl_path_equals_plain_learner(algo, precision):
    """comm_mode 2: the sharded code path (partials -> contiguous reduce -> in-graph ncclAllReduce over a
    one-rank communicator -> Adam from the reduced buffer) gives bit-identical results to the plain path."""
    o, m, h, L, B, C = 22, 6, 256, 2, 2048, 20_000
    g, _ = make_rings(o, m, C)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    plain = make_learner(g, p, algo, precision, h, L, B)
    nccl = make_learner(g, p, algo, precision, h, L, B, comm_mode=2)
    s1 = plain.update(B, 4)
    s2 = nccl.update(B, 4)
    for n in ("actor", "q1", "q2", "q1_targ"):
        assert np.array_equal(plain.get(n), nccl.get(n)), n
    assert s1["critic_loss"] == s2["critic_loss"]
