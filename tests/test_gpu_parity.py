"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle.

Bar (BASELINE.json north_star): replay indices and gathered rows
bit-exact; losses and every parameter / Adam-moment tensor after K updates within
||x - x*|| / ||x*|| <= 1e-4 (FP32 path) or 2e-2 (BF16 tensor-core path).
"""

import numpy as np
import pytest

import synthdata
from oracle import ring as oring, sac as osac, td3 as otd3

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_06126_b200 import spz  # noqa: E402

from tests.parity import TOL, make_rings, rel, run_parity  # noqa: E402,F401


def assert_update_direction(gpu_new, gpu_old, ref_new, ref_old, tag, cos_min=0.9, norm_tol=0.25):
    """The K-step parameter change on the GPU against the oracle's: the same direction (cosine) and size --
    a path that never updated (change 0) or updated a wrong way fails it, whatever the parameter bar says."""
    dg = np.asarray(gpu_new, np.float64) - np.asarray(gpu_old, np.float64)
    dr = np.asarray(ref_new, np.float64) - np.asarray(ref_old, np.float64)
    cos = float(dg @ dr / max(np.linalg.norm(dg) * np.linalg.norm(dr), 1e-300))
    ratio = float(np.linalg.norm(dg) / max(np.linalg.norm(dr), 1e-300))
    assert cos >= cos_min and abs(ratio - 1) <= norm_tol, (tag, "update direction", cos, ratio)


# ----------------------------------------------------------------------------- a1 + a2 bit-exact

@pytest.mark.parametrize("o,m,C,n_push,B", [
    (3, 1, 10_000, None, 256),        # PEN
    (3, 1, 100, 1, 1),                # fill 1, batch 1
    (22, 6, 5000, 3000, 1000),        # partial fill, ragged batch
    (44, 17, 4096, 10_000, 777),      # wrapped ring (10000 pushes into 4096 slots), odd batch
    (28, 8, 1_000_000, None, 32768),  # ANT-size ring, full batch
])
def test_replay_sample_bit_exact(o, m, C, n_push, B):
    g, r = make_rings(o, m, C, n_push)
    for step in (0, 7):
        idx = torch.empty(B, dtype=torch.int32, device="cuda")
        obs = torch.empty(B, o, device="cuda")
        act = torch.empty(B, m, device="cuda")
        rew = torch.empty(B, device="cuda")
        nobs = torch.empty(B, o, device="cuda")
        done = torch.empty(B, device="cuda")
        spz.spz_replay_sample(g.h, B, synthdata.SAMPLE_SEED, step, idx, obs, act, rew, nobs, done)
        ridx, rb = r.sample(B, synthdata.SAMPLE_SEED, step)
        assert np.array_equal(idx.cpu().numpy(), ridx)
        for name, t in (("obs", obs), ("act", act), ("rew", rew), ("next_obs", nobs), ("done", done)):
            assert np.array_equal(t.cpu().numpy(), rb[name]), name


def test_replay_errors_and_info():
    g = spz.Replay(3, 1, 8)
    assert g.info() == (0, 0, 8)
    with pytest.raises(spz.SpzError) as e:
        spz.spz_replay_sample(g.h, 1, 1, 0)
    assert e.value.status == spz.SPZ_ENODATA
    tr = synthdata.transitions("pendulum", 3, 1, 11)
    assert g.push(**tr) == 0
    assert g.info() == (11, 8, 8)


def test_replay_push_from_device_matches_host():
    o, m, C = 22, 6, 1000
    tr = synthdata.transitions("locomotion", o, m, 1500)
    a, b = spz.Replay(o, m, C), spz.Replay(o, m, C)
    a.push(**tr)
    b.push(**{k: torch.from_numpy(v).cuda() for k, v in tr.items()}, src_on_device=True)
    B = 512
    outs = []
    for g in (a, b):
        idx = torch.empty(B, dtype=torch.int32, device="cuda")
        obs = torch.empty(B, o, device="cuda")
        spz.spz_replay_sample(g.h, B, 5, 3, idx, obs)
        outs.append((idx.cpu().numpy(), obs.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_replay_push_pinned_matches_pageable():
    """Page-locked host fields take the DMA + device-pack path; the ring must be bit-identical to the
    host-pack path, including a push that wraps and one longer than the capacity."""
    o, m, C = 17, 5, 700
    rings = []
    for pinned in (False, True):
        g = spz.Replay(o, m, C)
        for n, seed in ((500, 1), (450, 2), (1600, 3)):
            tr = synthdata.transitions("locomotion", o, m, n, seed=seed)
            if pinned:
                tr = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in tr.items()}
            g.push(**tr)
        rings.append(g)
    assert rings[0].info() == rings[1].info()
    B = 700
    outs = []
    for g in rings:
        bufs = [torch.empty(B, dtype=torch.int32, device="cuda"), torch.empty(B, o, device="cuda"),
                torch.empty(B, m, device="cuda"), torch.empty(B, device="cuda"), torch.empty(B, o, device="cuda"),
                torch.empty(B, device="cuda")]
        spz.spz_replay_sample(g.h, B, 9, 4, *bufs)
        outs.append([b.cpu().numpy() for b in bufs])
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def test_update_async_overlapped_pushes_bit_identical():
    """push(k+1) issued while update k runs (spz_update_async / spz_update_wait) gives bit-identical
    parameters and statistics to the synchronous push, update sequence (device-side ordering of the
    ring writes after the in-flight reads); pinned and pageable pushes."""
    o, m, C, B, K = 22, 6, 3000, 1024, 6
    fresh = [synthdata.transitions("locomotion", o, m, B, seed=100 + k) for k in range(K)]
    res = []
    for mode in ("sync", "async_pinned", "async_pageable", "async2"):
        g, _ = make_rings(o, m, C)
        lrn = spz.Learner(g, precision="bf16", hidden=64, n_hidden=2, max_batch=B)
        stats = []
        for k in range(K):
            tr = fresh[k]
            if mode == "async_pinned":
                tr = {n: torch.from_numpy(v).pin_memory().numpy() for n, v in tr.items()}
            if mode == "sync":
                g.push(**tr)
                stats.append(lrn.update(B, 1))
            elif mode == "async2":  # two updates in flight: push k while k-2 and k-1 run
                g.push(**tr)
                if k >= 2:
                    stats.append(lrn.wait())
                lrn.update_async(B, 1)
            else:
                if k > 0:
                    g.push(**tr)  # overlaps update k-1 on the GPU
                    stats.append(lrn.wait())
                else:
                    g.push(**tr)
                lrn.update_async(B, 1)
        if mode == "async2":
            stats.append(lrn.wait())
            stats.append(lrn.wait())
        elif mode != "sync":
            stats.append(lrn.wait())
        res.append((stats, [lrn.get(n) for n in ("actor", "q1", "q2", "q1_targ")]))
    for other in res[1:]:
        assert other[0] == res[0][0]
        for a, b in zip(other[1], res[0][1]):
            assert np.array_equal(a, b)


# ----------------------------------------------------------------------------- whole update parity

@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_sac_parity_pendulum(precision):
    # BASELINE config 0: Pendulum-shaped SAC, 2x64, B 256, 10K ring (200 updates in the bench; 30 here)
    run_parity("sac", precision, 3, 1, 64, 2, 256, 10_000, 30, kind="pendulum")


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_sac_parity_ragged_multitile(precision):
    # several 128-row tiles plus a ragged tail; K tails (o + m = 28 not a multiple of 8/16/64)
    run_parity("sac", precision, 22, 6, 256, 2, 1000, 20_000, 5)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_td3_parity(precision):
    run_parity("td3", precision, 44, 17, 128, 3, 600, 8000, 4)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_sac_parity_wide_humanoid_shape(precision):
    # HUM shapes (o 44, m 17, 3x512): two 256-column tiles per hidden row (split row-dot partials)
    run_parity("sac", precision, 44, 17, 512, 3, 700, 8000, 3)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_td3_parity_wide_1024(precision):
    # TD3 config shapes (3x1024): four row-dot partials; steps 0..3 (two delayed actor updates).  Round 1 cut fp32
    # to 2 steps; with the kernel's decisions on both sides (reading #25) the 4-step fp32 run holds 1e-4.
    run_parity("td3", precision, 44, 17, 1024, 3, 520, 6000, 4)


@pytest.mark.parametrize("B", [4096, 10000])
def test_sac_parity_pair_schedule_critic_forward(B, monkeypatch):
    """The two-blocks-in-flight critic forward (default at >= 4 row blocks per CTA) forced at sizes where
    CTAs get 2..4 blocks: full pairs, a trailing single block, ragged last block."""
    monkeypatch.setenv("SPZ_MLP_PAIR", "1")
    run_parity("sac", "bf16", 22, 6, 256, 2, B, 20_000, 2)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("h,L,B", [(64, 2, 256), (256, 2, 1000)])
def test_ddpg_parity(precision, h, L, B):
    """DDPG (f4) on the TD3 kernels with the twin critic tied to the first, against oracle/ddpg.py (one
    critic).  Also: the twin stays bit-identical to the first critic, and setting it directly is refused."""
    from oracle import ddpg as oddpg
    o, m, C, K = 22, 6, 6000, 4
    g, r = make_rings(o, m, C)
    p = synthdata.init_params(o, m, h, L, algo="td3")
    lrn = spz.Learner(g, algo="ddpg", precision=precision, hidden=h, n_hidden=L, max_batch=B)
    lrn.set("actor", p["actor"])
    lrn.set("actor_targ", p["actor"])
    lrn.set("q1", p["q1"])
    lrn.set("q1_targ", p["q1"])
    with pytest.raises(spz.SpzError) as e:
        lrn.set("q2", p["q2"])
    assert e.value.status == spz.SPZ_EINVAL
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=False, td3_policy_delay=1,
                      td3_noise=0.0, td3_noise_clip=0.0)
    st = osac.State.create(p["actor"], p["q1"], p["q1"], log_alpha=0.0, actor_targ=p["actor"])
    tol = TOL[precision]
    for k in range(K):
        gs = lrn.update(B, 1)
        st, os_, _ = oddpg.ddpg_step(st, r, B, synthdata.SAMPLE_SEED, cfg)
        for key in ("critic_loss", "actor_loss", "q1_mean"):
            ref = os_[key]
            scale = max(abs(ref), os_.get(key + "_abs", 0.0))
            assert abs(gs[key] - ref) <= tol * max(scale, 1e-6) + (tol * 1e-2 if key == "q1_mean" else 0), (k, key, gs[key], ref)
    for n in ("actor", "q1", "q1_targ", "actor_targ"):
        assert rel(lrn.get(n), getattr(st, n)) <= tol, n
    for n in ("actor", "q1"):
        assert_update_direction(lrn.get(n), p[n], getattr(st, n), p[n], f"ddpg-{precision}-{n}")
    assert np.array_equal(lrn.get("q1"), lrn.get("q2")) and np.array_equal(lrn.get("q1_targ"), lrn.get("q2_targ"))
    c = lrn.counters()
    assert c["step"] == K and c["t_critic"] == K and c["t_actor"] == K


def test_sac_parity_graph_vs_eager_bit_identical():
    outs = []
    for use_graph in (True, False):
        g, _ = make_rings(5, 2, 3000)
        lrn = spz.Learner(g, precision="bf16", hidden=64, n_hidden=2, max_batch=512, use_graph=use_graph)
        lrn.update(512, 3)
        outs.append([lrn.get(n) for n in ("actor", "q1", "q2", "q1_targ")])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_determinism_two_runs_bit_identical():
    outs = []
    for _ in range(2):
        g, _ = make_rings(22, 6, 20_000)
        lrn = spz.Learner(g, precision="bf16", hidden=256, n_hidden=2, max_batch=2048)
        s = lrn.update(2048, 4)
        outs.append((s, [lrn.get(n) for n in ("actor", "q1", "q2")]))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


# ----------------------------------------------------------------------------- full-size configs (bench launch config)
# BASELINE.json configs 1-4 at full size, in the launch configuration bench.py times: raw gradients of every
# tensor at every step (k >= 1 included), Adam m and v, parameters, and the Adam / Polyak identities.

@pytest.fixture(scope="module")
def walker_rings():
    return make_rings(22, 6, 1_000_000)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_walker_full_size(precision, walker_rings):
    """Config 1: WLK, B 8192, 2x256, 1M ring."""
    run_parity("sac", precision, 22, 6, 256, 2, 8192, 1_000_000, 3, rings=walker_rings, tag=f"walker-{precision}")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_ant_full_size(precision):
    """Config 2 shapes on one GPU: ANT, o 28, m 8, B 32768 (> 148*128 rows: the GEMM + head-kernel actor
    backward), 2x256, 1M ring."""
    run_parity("sac", precision, 28, 8, 256, 2, 32768, 1_000_000, 2, tag=f"ant-{precision}")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_humanoid_full_size(precision):
    """Config 3 shapes on one GPU: HUM, B 65536, 3x512, 1M ring."""
    run_parity("sac", precision, 44, 17, 512, 3, 65536, 1_000_000, 2, tag=f"humanoid-{precision}")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_td3_full_size(precision):
    """Config 4 shapes on one GPU: TD3, B 131072, 3x1024, 4M ring; step 0 critic only, step 1 with the
    delayed actor, Polyak on all targets."""
    run_parity("td3", precision, 44, 17, 1024, 3, 131072, 4_000_000, 2, tag=f"td3-{precision}")


# mutation check: each of these breaks one piece of a6-a9 at the WLK launch configuration; the parity run
# must fail under every one (SPZ_DIAG_SKIP_OPS / SPZ_DIAG_MUTATE are diagnostics-only plan edits)
@pytest.mark.parametrize("env,val", [
    ("SPZ_DIAG_SKIP_OPS", "adam_polyak"),   # no optimizer step at all
    ("SPZ_DIAG_MUTATE", "tau0"),            # Polyak averaging dropped (targets frozen)
    ("SPZ_DIAG_MUTATE", "drop_wgrad=0"),    # q1 layer-0 weight gradient never computed
    ("SPZ_DIAG_MUTATE", "drop_wgrad=4"),    # q1 head weight gradient
    ("SPZ_DIAG_MUTATE", "drop_wgrad=8"),    # actor head weight gradient
    ("SPZ_DIAG_MUTATE", "drop_bias=3"),     # q2 layer-1 bias gradient
    ("SPZ_DIAG_SKIP_OPS", "actor_bwd_fused"),  # actor backward (a7) dropped
])
def test_mutation_fails_parity(env, val, walker_rings, monkeypatch):
    monkeypatch.setenv(env, val)
    with pytest.raises(AssertionError):
        run_parity("sac", "bf16", 22, 6, 256, 2, 8192, 1_000_000, 2, rings=walker_rings, tag=f"mutant-{val}")


# ----------------------------------------------------------------------------- API behaviour

def test_update_errors_and_batch_change():
    g, _ = make_rings(3, 1, 300, kind="pendulum")
    lrn = spz.Learner(g, precision="bf16", hidden=64, n_hidden=2, max_batch=256)
    with pytest.raises(spz.SpzError) as e:
        lrn.update(512, 1)
    assert e.value.status == spz.SPZ_EINVAL
    lrn.update(256, 2)
    lrn.update(100, 2)  # batch may change between calls; Adam moments preserved
    assert lrn.counters()["step"] == 4
    small = spz.Replay(3, 1, 100)
    small.push(**synthdata.transitions("pendulum", 3, 1, 10))
    l2 = spz.Learner(small, precision="bf16", hidden=64, n_hidden=2, max_batch=256)
    with pytest.raises(spz.SpzError) as e:
        l2.update(64, 1)
    assert e.value.status == spz.SPZ_ENODATA
    assert l2.counters()["step"] == 0


def test_set_get_roundtrip_and_default_init():
    g, _ = make_rings(22, 6, 2000)
    lrn = spz.Learner(g, precision="fp32", hidden=256, n_hidden=2, max_batch=1024)
    a = lrn.get("actor")
    # W, b ~ U(+-1/sqrt(fan_in)): first layer fan_in = 22
    W1 = a[:256 * 22]
    assert np.abs(W1).max() <= 1 / np.sqrt(22) + 1e-7 and abs(W1.mean()) < 0.01 and W1.std() > 0.1
    assert np.array_equal(lrn.get("q1"), lrn.get("q1_targ"))
    v = np.random.default_rng(0).standard_normal(a.size).astype(np.float32)
    lrn.set("actor", v)
    assert np.array_equal(lrn.get("actor"), v)
    assert abs(float(lrn.get("log_alpha")[0]) - np.log(0.2)) < 1e-6


def test_sync_actor_versioned_payload():
    g, _ = make_rings(22, 6, 2000)
    lrn = spz.Learner(g, precision="bf16", hidden=64, n_hidden=2, max_batch=512)
    n = lrn.get("actor").size
    buf = torch.zeros(spz.sync_bytes(n), dtype=torch.uint8, device="cuda")
    v1 = spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), buf.numel())
    lrn.update(512, 1)
    v2 = spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), buf.numel())
    assert v2 == v1 + 1
    hdr = buf[:spz.SYNC_HEADER_BYTES].cpu().numpy().view(np.uint64)
    # header: version, n_floats, seq of slot 0 / 1 (2v once version v in slot v & 1 is complete)
    assert hdr[0] == v2 and hdr[1] == n and hdr[2 + (v2 & 1)] == 2 * v2 and hdr[2 + (v1 & 1)] == 2 * v1
    off = spz.SYNC_HEADER_BYTES + (v2 & 1) * spz.sync_slot_bytes(n)
    assert np.array_equal(buf[off:off + 4 * n].cpu().numpy().view(np.float32), lrn.get("actor"))
    with pytest.raises(spz.SpzError) as e:  # too small for the two slots
        spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), 16 + 4 * n)
    assert e.value.status == spz.SPZ_EINVAL


def test_profile_and_launch_count():
    g, _ = make_rings(22, 6, 20_000)
    lrn = spz.Learner(g, precision="bf16", hidden=256, n_hidden=2, max_batch=8192)
    prof = lrn.profile(8192, 3)
    assert "gather" in prof and "adam_polyak" in prof and all(v > 0 for v in prof.values())
    # gather, 2 fused forwards, loss, critic dgrad, fused actor backward, wgrad, Adam (+ unfused variants)
    assert 8 <= lrn.launches_per_step(8192) <= 16
    assert lrn.counters()["step"] == 3


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("o,m,h,L,B,auto", [(22, 6, 64, 2, 256, False), (22, 6, 256, 2, 1000, False),
                                            (44, 17, 512, 3, 700, True)])
def test_sacv1_parity(precision, o, m, h, L, B, auto):
    """SAC v1 (f4: state-value network V + Polyak target V', no target critics) against oracle/sacv1.py:
    fused value forward (h <= 256) or the GEMM path (h = 512), loss-kernel g_V, value dgrad / wgrad in the
    critics' launches, Adam + Polyak on V'.  Fixed temperature (v1's default) and learned (auto)."""
    from oracle import sacv1 as ov1
    C, K = 6000, 3
    g, r = make_rings(o, m, C)
    p = synthdata.init_params(o, m, h, L, algo="sacv1")
    lrn = spz.Learner(g, algo="sacv1", precision=precision, hidden=h, n_hidden=L, max_batch=B, alpha_auto=int(auto))
    for n in ("actor", "q1", "q2", "v"):
        lrn.set(n, p[n])
    lrn.set("v_targ", 0.5 * p["v"])  # a target that differs from V, so y_Q really reads V'
    for absent in ("q1_targ", "q2_targ", "actor_targ"):
        with pytest.raises(spz.SpzError):
            lrn.get(absent)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=auto)
    la = float(lrn.get("log_alpha")[0])
    st = ov1.State.create(p["actor"], p["q1"], p["q2"], p["v"], v_targ=0.5 * p["v"], log_alpha=la)
    tol = TOL[precision]
    for k in range(K):
        gs = lrn.update(B, 1)
        st, os_, _ = ov1.sacv1_step(st, r, B, synthdata.SAMPLE_SEED, cfg)
        assert gs["step"] == k + 1
        for key in ("critic_loss", "value_loss", "actor_loss", "q1_mean", "q2_mean", "logp_mean", "alpha"):
            ref = os_[key]
            scale = max(abs(ref), os_.get(key + "_abs", 0.0))
            assert abs(gs[key] - ref) <= tol * max(scale, 1e-6) + (tol * 1e-2 if key in ("q1_mean", "q2_mean") else 0), (k, key, gs[key], ref)
    for n in ("actor", "q1", "q2", "v", "v_targ"):
        assert rel(lrn.get(n), getattr(st, n)) <= tol, (n, rel(lrn.get(n), getattr(st, n)))
    for n in ("actor", "q1", "q2", "v"):
        assert_update_direction(lrn.get(n), p[n], getattr(st, n), p[n], f"sacv1-{precision}-{n}")
    assert rel(lrn.get("v", spz.SPZ_S_ADAM_M), st.opt["v"].m) <= 10 * tol
    assert abs(float(lrn.get("log_alpha")[0]) - st.log_alpha) <= tol * max(1.0, abs(st.log_alpha))
    if not auto:
        assert float(lrn.get("log_alpha")[0]) == la
    c = lrn.counters()
    assert c["step"] == K and c["t_critic"] == K and c["t_actor"] == K and c["t_alpha"] == (K if auto else 0)


def test_sacv1_graph_eager_async_bit_identical():
    """SAC v1: the graph replay, the eager launches and two updates in flight give bit-identical parameters."""
    outs = []
    for mode in ("graph", "eager", "async"):
        g, _ = make_rings(7, 3, 3000)
        lrn = spz.Learner(g, algo="sacv1", precision="bf16", hidden=64, n_hidden=2, max_batch=512,
                          use_graph=(mode != "eager"))
        if mode == "async":
            for _ in range(3):
                lrn.update_async(512, 1)
            lrn.wait()
            lrn.wait()
            lrn.wait()
        else:
            lrn.update(512, 3)
        outs.append([lrn.get(n) for n in ("actor", "q1", "q2", "v", "v_targ")])
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_wide_observation_376(precision):
    """A MuJoCo Humanoid-v4-sized observation (o 376, m 17: 2o + m + 2 = 771-float records, 98 KB of gather
    staging per block -- past the 48 KB default): replay sampling stays bit-exact and the update (per-layer
    GEMM path for a K = 376 first layer) matches the oracle."""
    o, m, C, B = 376, 17, 3000, 300
    g, r = make_rings(o, m, C)
    idx = torch.empty(B, dtype=torch.int32, device="cuda")
    obs = torch.empty(B, o, device="cuda")
    nobs = torch.empty(B, o, device="cuda")
    spz.spz_replay_sample(g.h, B, synthdata.SAMPLE_SEED, 3, idx, obs, None, None, nobs)
    ridx, rb = r.sample(B, synthdata.SAMPLE_SEED, 3)
    assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(obs.cpu().numpy(), rb["obs"])
    assert np.array_equal(nobs.cpu().numpy(), rb["next_obs"])
    run_parity("sac", precision, o, m, 128, 2, B, C, 2, rings=(g, r), tag=f"obs376-{precision}")


def test_oversized_record_rejected():
    with pytest.raises(spz.SpzError) as e:
        spz.Replay(1000, 17, 100)  # 2017-float records: past the 227 KB gather staging
    assert e.value.status == spz.SPZ_EUNSUPPORTED


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("o,m,B", [(22, 6, 1000), (3, 1, 256), (44, 17, 777), (44, 17, 30000), (400, 17, 20000)])
def test_learner_gather_operands_bit_exact(precision, o, m, B):
    """a1-a2 inside the update: the step's indices equal the oracle's, and the gathered operands are
    exactly the sampled records rounded once to the operand type (bf16 RNE / fp32), with every padding
    column zero (written once at allocation, never by the 128-bit vector stores).  B 30000 / 20000: more
    32-row groups than 4 blocks per SM, so blocks walk several groups -- double-buffered asynchronous record
    copies (44-float observations), single buffer (400: two 105 KB buffers do not fit)."""
    g, r = make_rings(o, m, max(5000, B))
    lrn = spz.Learner(g, precision=precision, hidden=64, n_hidden=2, max_batch=B)
    for k in range(2):
        lrn.update(B, 1)
        ridx, rb = r.sample(B, synthdata.SAMPLE_SEED, k)
        assert np.array_equal(lrn.debug("idx")[:B], ridx)
        rnd = (lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).float().numpy()) \
            if precision == "bf16" else (lambda x: x)
        Xa = lrn.debug("Xa")
        lda = Xa.size // (2 * B)
        Xa = Xa.reshape(2 * B, lda)
        assert np.array_equal(Xa[:B, :o], rnd(rb["next_obs"])) and np.array_equal(Xa[B:, :o], rnd(rb["obs"]))
        assert not Xa[:, o:].any()
        Xc = lrn.debug("Xc")
        ldc = Xc.size // (3 * B)
        Xc = Xc.reshape(3 * B, ldc)
        assert np.array_equal(Xc[:B, :o], rnd(rb["obs"])) and np.array_equal(Xc[:B, o:o + m], rnd(rb["act"]))
        assert np.array_equal(Xc[B:2 * B, :o], rnd(rb["obs"])) and np.array_equal(Xc[2 * B:, :o], rnd(rb["next_obs"]))
        assert not Xc[:, o + m:].any()
        assert np.array_equal(lrn.debug("r")[:B], rb["rew"]) and np.array_equal(lrn.debug("d")[:B], rb["done"])


@pytest.mark.parametrize("algo,precision,B", [("sac", "bf16", 2048), ("sac", "fp32", 512), ("td3", "bf16", 2048),
                                              ("sac", "bf16", 40000)])
def test_nonfinite_loss_halts_before_the_step(algo, precision, B):
    """A non-finite loss (NaN rewards in the ring) halts the learner at the state before the failing step
    (SPEC S:68): SPZ_ENONFINITE from that update, every trained tensor unchanged, the step counter not
    advanced, and every later update refused -- with the loss totals deferred to the optimizer (its blocks decide
    from the loss kernel's non-finite flag word) as with the in-kernel reduction (B 40000: one block per row group
    past the resident grid)."""
    o, m, C = 22, 6, 50_000
    g = spz.Replay(o, m, C)
    tr = synthdata.transitions("locomotion", o, m, C)
    g.push(**tr)
    lrn = spz.Learner(g, algo=algo, precision=precision, hidden=256, n_hidden=2, max_batch=B)
    lrn.update(B, 2)
    before = [lrn.get(n) for n in ("actor", "q1", "q2", "q1_targ")]
    step0 = lrn.counters()["step"]
    bad = dict(tr)
    bad["rew"] = np.array(tr["rew"], copy=True)
    bad["rew"][::7] = np.nan  # every 7th transition: sampled in any batch of this size
    g2 = spz.Replay(o, m, C)
    g2.push(**bad)
    lrn2 = spz.Learner(g2, algo=algo, precision=precision, hidden=256, n_hidden=2, max_batch=B)
    for name, v in zip(("actor", "q1", "q2", "q1_targ"), before):
        lrn2.set(name, v)
    with pytest.raises(spz.SpzError) as e:
        lrn2.update(B, 1)
    assert e.value.status == spz.SPZ_ENONFINITE
    for name, v in zip(("actor", "q1", "q2", "q1_targ"), before):
        assert np.array_equal(lrn2.get(name), v), name
    assert lrn2.counters()["step"] == 0
    with pytest.raises(spz.SpzError) as e2:
        lrn2.update(B, 1)
    assert e2.value.status == spz.SPZ_ENONFINITE
    assert step0 == 2
