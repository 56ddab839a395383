"""World-size-2 gloo tests of the multi-process plumbing (CPU, no GPU needed)."""

import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_06126_b200.dist import broadcast_bytes, max_over_ranks, row_shard, sum_over_ranks


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = bytes(range(128)) if rank == 0 else None
    got = broadcast_bytes(uid)
    mx = max_over_ranks(1.5 + rank)
    sm = sum_over_ranks(row_shard(8192, world, rank)[1])
    q.put((rank, got == bytes(range(128)), mx, sm))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_broadcast_and_reductions(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res)
    assert all(mx == 1.5 + world - 1 for _, _, mx, _ in res)
    assert all(sm == 8192 for _, _, _, sm in res)


def test_row_shard_partition_matches_oracle_schedule():
    from oracle.schedules import _shards
    for B in (1, 7, 256, 8192, 8193):
        for W in (1, 2, 3, 8):
            if B < W:
                continue
            mine = [row_shard(B, W, r) for r in range(W)]
            assert mine == _shards(B, W)
            assert sum(n for _, n in mine) == B


# ----------------------------------------------------------------------------- the learner's host-side plan, world 2

def _plan_worker(rank, world, port, q, algo, mode):
    """One rank of a world-2 group: its partition / role from the C library's spz_plan_rank (the learner's
    own plan), its share of the step in the float64 oracle, the exchange over gloo, and the result."""
    import numpy as np
    import torch
    import synthdata
    from oracle import ring as oring, sac as osac, td3 as otd3
    from paper_2312_06126_b200 import spz
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o, m, h, L, B, C = 5, 2, 16, 2, 37, 300
    tr = synthdata.transitions("locomotion", o, m, C)
    ring = oring.Ring(o, m, C)
    ring.push(**tr)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=algo == "sac")
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=np.log(0.2),
                           actor_targ=p["actor"] if algo == "td3" else None)
    seed, out = synthdata.SAMPLE_SEED, {}
    if mode == "dp":
        plan = spz.spz_plan_rank(B, world, rank)
        for k in range(2):  # two steps: the second uses the first's (identical) state on every rank
            r0, n = plan["row0"], plan["rows"]
            idx, batch = ring.sample(n, seed, k, row0=r0, global_batch=B)
            if algo == "sac":
                eps, eps2 = osac.draw_noise(seed, k, n, m, row0=r0)
                g, sums = osac.sac_grads(st, batch, eps, eps2, cfg, B)
            else:
                g, sums = otd3.td3_grads(st, batch, otd3.draw_smoothing(seed, k, n, cfg, row0=r0), cfg, B, k)
            # the step's allreduce: [gradients | loss totals], SUM over the group (global 1/B: exact)
            for key in sorted(g):
                t = torch.from_numpy(np.array(g[key], np.float64))
                dist.all_reduce(t)
                g[key] = t.numpy()
            tot = torch.tensor([sums[k2] for k2 in ("lq", "q1", "q2")], dtype=torch.float64)
            dist.all_reduce(tot)
            st = osac.sac_apply(st, g, cfg) if algo == "sac" else otd3.td3_apply(st, g, cfg, k)
            out[f"lq{k}"] = float(tot[0])
    else:  # split: rank 0 critic group, rank 1 actor group
        role = spz.SPZ_ROLE_CRITIC if rank == 0 else spz.SPZ_ROLE_ACTOR
        plan = spz.spz_plan_rank(B, world, rank, role=role, n_critic_ranks=1)
        k = 0
        idx, batch = ring.sample(B, seed, k, row0=plan["row0"], global_batch=B)
        eps, eps2 = osac.draw_noise(seed, k, B, m)
        critic = plan["role"] == spz.SPZ_ROLE_CRITIC
        g, sums = osac.sac_grads(st, batch, eps, eps2, cfg, B, critic=critic, actor=not critic)
        st = osac.sac_apply(st, g, cfg, critic=critic, actor=not critic)
        # a10: broadcast phi (+ log alpha) from the actor root and theta from the critic root
        ta = torch.from_numpy(np.concatenate([st.actor, [st.log_alpha]]))
        dist.broadcast(ta, src=plan["actor_root"])
        tq = torch.from_numpy(np.concatenate([st.q1, st.q2]))
        dist.broadcast(tq, src=plan["critic_root"])
        st.actor, st.log_alpha = ta.numpy()[:-1].copy(), float(ta.numpy()[-1])
        st.q1, st.q2 = tq.numpy()[:st.q1.size].copy(), tq.numpy()[st.q1.size:].copy()
    out.update(plan=plan, actor=st.actor, q1=st.q1, q2=st.q2, q1_targ=st.q1_targ, log_alpha=st.log_alpha)
    q.put((rank, out))
    dist.destroy_process_group()


def _run_world2(algo, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000 + (7 if mode == "split" else 0) + (3 if algo == "td3" else 0)
    ps = [ctx.Process(target=_plan_worker, args=(r, 2, port, q, algo, mode)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("algo", ["sac", "td3"])
def test_world2_row_sharded_plan_equals_single(algo):
    """dp, world 2: the C plan's shards tile [0, B) (ragged B = 37), the SUM-allreduced shard gradients and
    loss totals give exactly the single-device step (1e-12), and both ranks hold bit-identical parameters."""
    import numpy as np
    import synthdata
    from oracle import ring as oring, sac as osac, td3 as otd3
    res = _run_world2(algo, "dp")
    plans = sorted((res[r]["plan"]["row0"], res[r]["plan"]["rows"]) for r in (0, 1))
    assert plans == [(0, 19), (19, 18)]
    o, m, h, L, B, C = 5, 2, 16, 2, 37, 300
    ring = oring.Ring(o, m, C)
    ring.push(**synthdata.transitions("locomotion", o, m, C))
    p = synthdata.init_params(o, m, h, L, algo=algo)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=algo == "sac")
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=np.log(0.2),
                           actor_targ=p["actor"] if algo == "td3" else None)
    for k in range(2):
        st, stats, _ = (osac.sac_step if algo == "sac" else otd3.td3_step)(st, ring, B, synthdata.SAMPLE_SEED, cfg)
        assert abs(res[0][f"lq{k}"] / B - stats["critic_loss"]) <= 1e-12 * abs(stats["critic_loss"])
    for n in ("actor", "q1", "q2", "q1_targ"):
        assert np.array_equal(res[0][n], res[1][n]), n  # replicated optimizer: identical on every rank
        ref = getattr(st, n)
        assert np.linalg.norm(res[0][n] - ref) <= 1e-12 * np.linalg.norm(ref), n


def test_world2_split_plan_exchange_equals_single():
    """split, world 2 (rank 0 critic group, rank 1 actor group from the C plan): each computes its half of the
    Jacobi step, the a10 broadcast from the plan's roots exchanges phi / log alpha and theta, and both ranks
    then hold exactly the single-device step's parameters."""
    import numpy as np
    import synthdata
    from oracle import ring as oring, sac as osac
    res = _run_world2("sac", "split")
    assert res[0]["plan"]["role"] == 1 and res[1]["plan"]["role"] == 2
    assert res[0]["plan"]["actor_root"] == 1 and res[0]["plan"]["critic_root"] == 0
    o, m, h, L, B, C = 5, 2, 16, 2, 37, 300
    ring = oring.Ring(o, m, C)
    ring.push(**synthdata.transitions("locomotion", o, m, C))
    p = synthdata.init_params(o, m, h, L)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L)
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=np.log(0.2))
    st, _, _ = osac.sac_step(st, ring, B, synthdata.SAMPLE_SEED, cfg)
    for r in (0, 1):
        for n in ("actor", "q1", "q2"):
            assert np.array_equal(res[r][n], getattr(st, n)), (r, n)
        assert res[r]["log_alpha"] == st.log_alpha
    assert np.array_equal(res[0]["q1_targ"], st.q1_targ)  # the critic group's Polyak


def test_bench_dry_run_gpus2_reports_partitions():
    """`bench.py --gpus 2 --dry-run` re-launches itself under torch.distributed.run (gloo, no GPU) and
    reports n_gpus 2 and each rank's plan from the C library."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for mode, scaling, GB in (("dp", "weak", 16384), ("dp", "strong", 8192), ("split", "strong", 8192)):
        p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--mode", mode, "--scaling", scaling],
                           cwd=root, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        line = json.loads(p.stdout.strip().splitlines()[-1])
        assert line["n_gpus"] == 2 and line["partitions_tile_batch"] and line["config"]["global_batch"] == GB
        rows = sorted((q["row0"], q["rows"]) for q in line["plans"])
        if mode == "dp":
            assert rows == [(0, GB // 2), (GB // 2, GB // 2)]
        else:  # each group (one rank) reads the whole batch
            assert rows == [(0, GB), (0, GB)] and {q["role"] for q in line["plans"]} == {1, 2}


def test_plan_rank_validation_and_partitions():
    """spz_plan_rank (host only, no GPU): bad layouts are rejected; partitions of every (B, G) tile [0, B) in rank
    order with the first B % G ranks one row longer (the oracle's schedule); split roles name the leaders."""
    from oracle.schedules import _shards
    from paper_2312_06126_b200 import spz
    with pytest.raises(spz.SpzError):
        spz.spz_plan_rank(100, 2, 2)                      # rank outside the world
    with pytest.raises(spz.SpzError):
        spz.spz_plan_rank(1, 2, 0)                        # fewer rows than ranks
    with pytest.raises(spz.SpzError):                     # rank 0 must be in the critic group
        spz.spz_plan_rank(100, 4, 0, role=spz.SPZ_ROLE_ACTOR, n_critic_ranks=2)
    with pytest.raises(spz.SpzError):
        spz.spz_plan_rank(100, 4, 3, role=spz.SPZ_ROLE_ACTOR, n_critic_ranks=4)  # no actor group left
    for B in (7, 8192, 8193, 131072):
        for G in (1, 2, 3, 8):
            if B < G:
                continue
            got = [spz.spz_plan_rank(B, G, r) for r in range(G)]
            assert [(p["row0"], p["rows"]) for p in got] == _shards(B, G)
            assert all(p["allreduce"] == (G > 1) and p["group_size"] == G for p in got)
    plans = [spz.spz_plan_rank(8192, 8, r, role=spz.SPZ_ROLE_CRITIC if r < 6 else spz.SPZ_ROLE_ACTOR,
                               n_critic_ranks=6) for r in range(8)]
    assert [p["group_size"] for p in plans] == [6] * 6 + [2] * 2
    assert [p["group_rank"] for p in plans] == list(range(6)) + [0, 1]
    assert all(p["actor_root"] == 6 and p["critic_root"] == 0 for p in plans)
    assert [(p["row0"], p["rows"]) for p in plans[6:]] == _shards(8192, 2)
