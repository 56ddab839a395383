"""Pins for oracle/sacv1.py (SAC v1 with a state-value network).

The v1 losses are pinned against an independent float64 torch.autograd implementation, and against
the (separately pinned) SAC oracle where the two methods coincide: the policy and temperature
gradients are SAC's, and the value target is SAC's soft Bellman target with s2 = s, r = 0, d = 0,
gamma = 1, targets = online critics and eps2 = eps.
"""

import numpy as np
import torch

import synthdata
from oracle import mlp, optim, philox, ring as oring, sac, sacv1


def small_problem(o=5, m=3, h=16, L=2, C=200, seed=0, alpha_auto=True):
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=alpha_auto)
    r = oring.Ring(o, m, C)
    r.push(**synthdata.transitions("locomotion", o, m, C, seed=seed + 1))
    p = synthdata.init_params(o, m, h, L, algo="sacv1", seed=seed)
    # a target V that differs from the online one, so the Q target really reads V_psibar
    st = sacv1.State.create(p["actor"], p["q1"], p["q2"], p["v"], v_targ=0.5 * p["v"], log_alpha=np.log(0.2))
    return cfg, r, st


def _torch_mlp(params, x):
    a = x
    for l, (W, b) in enumerate(params):
        a = torch.nn.functional.linear(a, W, b)
        if l < len(params) - 1:
            a = torch.relu(a)
    return a


def _tp(flat, shapes, grad):
    return [(torch.tensor(W, requires_grad=grad), torch.tensor(b, requires_grad=grad))
            for W, b in mlp.unflatten(flat, shapes)]


def test_sacv1_grads_match_torch_autograd():
    cfg, r, st = small_problem()
    B = 48
    idx, batch = r.sample(B, 6126, 0)
    eps = philox.normals(6126, 0, philox.S_EPS, B, cfg.act_dim)
    grads, sums = sacv1.sacv1_grads(st, batch, eps, cfg, B)

    ash, csh, vsh = sac.actor_shapes(cfg), sac.critic_shapes(cfg), sacv1.value_shapes(cfg)
    s, a, rr, s2, d = [torch.tensor(np.asarray(batch[k], np.float64)) for k in ("obs", "act", "rew", "next_obs", "done")]
    A = _tp(st.actor, ash, True)
    Q1, Q2 = _tp(st.q1, csh, True), _tp(st.q2, csh, True)
    V, Vt = _tp(st.v, vsh, True), _tp(st.v_targ, vsh, False)
    log_alpha = torch.tensor(st.log_alpha, dtype=torch.float64, requires_grad=True)
    m = cfg.act_dim
    H = _torch_mlp(A, s)
    mu, l = H[:, :m], H[:, m:]
    lc = torch.clamp(l, cfg.log_std_min, cfg.log_std_max)
    e = torch.tensor(eps)
    u = mu + torch.exp(lc) * e
    lpt = (-0.5 * e ** 2 - lc - 0.5 * np.log(2 * np.pi) - 2 * (np.log(2.0) - u - torch.nn.functional.softplus(-2 * u))).sum(1)
    at = torch.tanh(u)
    alpha = torch.exp(log_alpha).detach()
    det = lambda P: [(W.detach(), b.detach()) for W, b in P]
    with torch.no_grad():
        qmin = torch.minimum(_torch_mlp(Q1, torch.cat([s, at], 1))[:, 0], _torch_mlp(Q2, torch.cat([s, at], 1))[:, 0])
        y_v = qmin - alpha * lpt
        y = rr + cfg.gamma * (1 - d) * _torch_mlp(Vt, s2)[:, 0]
    LV = ((_torch_mlp(V, s)[:, 0] - y_v) ** 2).mean()
    LQ = ((_torch_mlp(Q1, torch.cat([s, a], 1))[:, 0] - y) ** 2 + (_torch_mlp(Q2, torch.cat([s, a], 1))[:, 0] - y) ** 2).mean()
    Lpi = (alpha * lpt - torch.minimum(_torch_mlp(det(Q1), torch.cat([s, at], 1))[:, 0],
                                       _torch_mlp(det(Q2), torch.cat([s, at], 1))[:, 0])).mean()
    La = -(log_alpha * (lpt.detach() + cfg.target_entropy)).mean()
    (LV + LQ + Lpi + La).backward()
    flat = lambda P: np.concatenate([np.concatenate([W.grad.numpy().ravel(), b.grad.numpy()]) for W, b in P])
    for key, P in (("q1", Q1), ("q2", Q2), ("v", V), ("actor", A)):
        assert np.allclose(grads[key], flat(P), rtol=1e-10, atol=1e-13), key
    assert np.isclose(grads["log_alpha"][0], log_alpha.grad.item(), rtol=1e-12)
    assert np.isclose(sums["lv"] / B, LV.item(), rtol=1e-12)
    assert np.isclose(sums["lq"] / B, LQ.item(), rtol=1e-12)
    assert np.isclose(sums["lpi"] / B, Lpi.item(), rtol=1e-12)


def test_policy_and_temperature_gradients_are_sacs():
    """v1 and v2 share L_pi and L_alpha: same batch, eps, actor, critics, alpha -> same gradients."""
    cfg, r, st = small_problem()
    B = 40
    _, batch = r.sample(B, 6126, 3)
    eps = philox.normals(6126, 3, philox.S_EPS, B, cfg.act_dim)
    g1, s1 = sacv1.sacv1_grads(st, batch, eps, cfg, B)
    st2 = sac.State.create(st.actor, st.q1, st.q2, log_alpha=st.log_alpha)
    g2, s2 = sac.sac_grads(st2, batch, eps, eps, cfg, B, critic=False, actor=True)
    assert np.array_equal(g1["actor"], g2["actor"])
    assert np.array_equal(g1["log_alpha"], g2["log_alpha"])
    assert s1["lpi"] == s2["lpi"] and s1["logp"] == s2["logp"]


def test_value_target_is_sacs_soft_bellman_target_at_s():
    """y_V = min Q(s, a~) - alpha log pi~ is SAC's y with s2 = s, r = 0, d = 0, gamma = 1, Q' = Q, eps2 = eps."""
    cfg, r, st = small_problem()
    B = 32
    _, batch = r.sample(B, 6126, 1)
    eps = philox.normals(6126, 1, philox.S_EPS, B, cfg.act_dim)
    _, s1 = sacv1.sacv1_grads(st, batch, eps, cfg, B)
    b2 = dict(batch)
    b2["next_obs"] = batch["obs"]
    b2["rew"] = np.zeros_like(batch["rew"])
    b2["done"] = np.zeros_like(batch["done"])
    cfg2 = sac.Config(obs_dim=cfg.obs_dim, act_dim=cfg.act_dim, hidden=cfg.hidden, n_hidden=cfg.n_hidden, gamma=1.0)
    st2 = sac.State.create(st.actor, st.q1, st.q2, log_alpha=st.log_alpha)
    _, s2 = sac.sac_grads(st2, b2, eps, eps, cfg2, B, critic=True, actor=False)
    assert np.allclose(s1["y_v"], s2["y"], rtol=1e-13, atol=1e-13)


def test_q_target_special_cases():
    """gamma = 0 or d = 1: y_Q = r exactly (V_psibar drops out); otherwise it reads the target V only."""
    cfg, r, st = small_problem()
    B = 24
    _, batch = r.sample(B, 6126, 2)
    eps = philox.normals(6126, 2, philox.S_EPS, B, cfg.act_dim)
    cfg.gamma = 0.0
    _, s0 = sacv1.sacv1_grads(st, batch, eps, cfg, B)
    assert np.array_equal(s0["y"], np.asarray(batch["rew"], np.float64))
    cfg.gamma = 0.99
    b1 = dict(batch)
    b1["done"] = np.ones_like(batch["done"])
    _, s1 = sacv1.sacv1_grads(st, b1, eps, cfg, B)
    assert np.array_equal(s1["y"], np.asarray(batch["rew"], np.float64))
    # changing the online V does not move y_Q; changing the target V does
    st_a = st.copy()
    st_a.v = st.v * 3.0
    _, sa = sacv1.sacv1_grads(st_a, batch, eps, cfg, B)
    _, sb = sacv1.sacv1_grads(st, batch, eps, cfg, B)
    assert np.array_equal(sa["y"], sb["y"])
    st_b = st.copy()
    st_b.v_targ = st.v_targ * 3.0
    _, sc = sacv1.sacv1_grads(st_b, batch, eps, cfg, B)
    assert not np.allclose(sc["y"], sb["y"])


def test_step_updates_value_target_by_polyak_and_keeps_alpha_fixed():
    cfg, r, st = small_problem(alpha_auto=False)
    st1, stats, _ = sacv1.sacv1_step(st, r, 48, 6126, cfg)
    assert np.allclose(st1.v_targ, cfg.tau * st1.v + (1 - cfg.tau) * st.v_targ, rtol=0, atol=1e-15)
    assert st1.log_alpha == st.log_alpha and st1.step == 1
    # the value net moved by exactly one Adam step of its gradient
    _, batch = r.sample(48, 6126, 0)
    eps = philox.normals(6126, 0, philox.S_EPS, 48, cfg.act_dim)
    g, _ = sacv1.sacv1_grads(st, batch, eps, cfg, 48)
    v_ref = optim.adam_step(st.v, g["v"], optim.AdamState(st.v.size), cfg.lr_critic, cfg.beta1, cfg.beta2, cfg.adam_eps)
    assert np.array_equal(st1.v, v_ref)
    assert stats["value_loss"] > 0 and np.isfinite(stats["critic_loss"])


def test_constant_value_net_gradient_closed_form():
    """V = c (every weight and bias zero but the output bias): dL_V/dc = (2/B) sum_j (c - y_V,j), every other
    V gradient zero (hidden activations relu(0) = 0, ReLU'(0) = 0)."""
    cfg, r, st = small_problem()
    B = 36
    _, batch = r.sample(B, 6126, 4)
    eps = philox.normals(6126, 4, philox.S_EPS, B, cfg.act_dim)
    c = 0.37
    st.v = np.zeros_like(st.v)
    st.v[-1] = c
    g, sums = sacv1.sacv1_grads(st, batch, eps, cfg, B)
    assert np.isclose(g["v"][-1], 2.0 / B * np.sum(c - sums["y_v"]), rtol=1e-13)
    assert np.count_nonzero(g["v"][:-1]) == 0
    assert np.isclose(sums["lv"], np.sum((c - sums["y_v"]) ** 2), rtol=1e-13)
