"""Pins for oracle/sac.py and oracle/td3.py (the update step itself)."""

import numpy as np
import pytest
import torch
from scipy import integrate

import synthdata
from oracle import mlp, ring as oring, sac, td3


def small_problem(algo="sac", o=5, m=3, h=16, L=2, C=200, seed=0):
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L)
    r = oring.Ring(o, m, C)
    r.push(**synthdata.transitions("locomotion", o, m, C, seed=seed + 1))
    p = synthdata.init_params(o, m, h, L, algo=algo, seed=seed)
    st = sac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=np.log(0.2),
                          actor_targ=p["actor"] if algo == "td3" else None)
    return cfg, r, st


# ----------------------------------------------------------------------------- head

def _linear_actor(mu, l, o=2):
    m = len(mu)
    W = np.zeros((2 * m, o))
    return [(W, np.concatenate([mu, l]))]


@pytest.mark.parametrize("mu,l", [(0.0, 0.0), (0.7, -0.5), (-1.3, 0.6), (2.5, -1.0)])
def test_logprob_normalises_quadrature(mu, l):
    # exp(log pi) integrates to 1 over the bounded action interval
    cfg = sac.Config(obs_dim=2, act_dim=1)
    A = _linear_actor(np.array([mu]), np.array([l]))
    sigma = np.exp(l)

    def logp_at_u(u):
        eps = np.atleast_1d((u - mu) / sigma).reshape(-1, 1)
        _, lp, _, _ = sac.policy_forward(A, np.zeros((eps.shape[0], 2)), eps, cfg)
        return lp

    # change of variable a = tanh(u): integrand exp(log pi(a)) (1 - tanh(u)^2)
    u = np.linspace(mu - 14 * sigma, mu + 14 * sigma, 200001)
    f = np.exp(logp_at_u(u)) * (1 - np.tanh(u) ** 2)
    assert abs(np.trapezoid(f, u) - 1.0) < 1e-8
    # a-space (density spikes near +-1 when sigma is large): within 1e-3
    val, _ = integrate.quad(lambda a: float(np.exp(logp_at_u(np.arctanh(a)))[0]), -1 + 1e-12, 1 - 1e-12, limit=400)
    assert abs(val - 1.0) < 1e-3


def test_deterministic_zero_mean_gives_zero_action():
    cfg = sac.Config(obs_dim=2, act_dim=3)
    A = _linear_actor(np.zeros(3), np.zeros(3))
    a, lp, _, _ = sac.policy_forward(A, np.zeros((4, 2)), np.zeros((4, 3)), cfg)
    assert np.array_equal(a, np.zeros((4, 3)))


def test_squash_term_finite_at_large_u():
    # reading #7: the stable form is finite where ln(1 - tanh^2 + 0) is -inf
    cfg = sac.Config(obs_dim=2, act_dim=1)
    A = _linear_actor(np.array([30.0]), np.array([-20.0]))
    _, lp, _, _ = sac.policy_forward(A, np.zeros((1, 2)), np.zeros((1, 1)), cfg)
    assert np.isfinite(lp).all()


def test_head_backward_vs_finite_differences():
    rng = np.random.default_rng(4)
    cfg = sac.Config(obs_dim=2, act_dim=4)
    B = 6
    mu = rng.normal(0, 2, (B, 4))
    mu[0, 0] = 19.0  # |u| ~ 20
    l = rng.uniform(-3, 1.5, (B, 4))
    l[1, 1] = -25.0  # below the clamp: no gradient
    l[2, 2] = 3.5  # above the clamp: no gradient
    eps = rng.standard_normal((B, 4))
    g_a = rng.standard_normal((B, 4))
    g_lp = rng.standard_normal(B)

    # use the oracle for the forward pieces: a row-wise linear actor with per-row bias is not
    # expressible, so evaluate the oracle head on one row at a time
    def oracle_obj(mu_, l_):
        tot = 0.0
        for j in range(B):
            A = _linear_actor(mu_[j], l_[j])
            a, lp, _, _ = sac.policy_forward(A, np.zeros((1, 2)), eps[j:j + 1], cfg)
            tot += np.sum(g_a[j] * a[0]) + g_lp[j] * lp[0]
        return tot

    heads = []
    dH = np.zeros((B, 8))
    for j in range(B):
        A = _linear_actor(mu[j], l[j])
        _, _, _, head = sac.policy_forward(A, np.zeros((1, 2)), eps[j:j + 1], cfg)
        dH[j] = sac.policy_head_backward(head, g_a[j:j + 1], g_lp[j:j + 1], cfg)[0]
    h = 1e-6
    for j in range(B):
        for q in range(4):
            for which in (0, 1):
                P = [mu.copy(), l.copy()]
                P[which][j, q] += h
                fp = oracle_obj(*P)
                P[which][j, q] -= 2 * h
                fm = oracle_obj(*P)
                fd = (fp - fm) / (2 * h)
                an = dH[j, which * 4 + q]
                assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd)), (j, q, which, fd, an)
    assert dH[1, 4 + 1] == 0.0 and dH[2, 4 + 2] == 0.0


def test_clamp_gradient_inclusive_at_bounds_like_torch():
    cfg = sac.Config(obs_dim=2, act_dim=2)
    l = np.array([[-20.0, 2.0]])
    mu = np.array([[0.3, -0.2]])
    eps = np.array([[0.5, -1.1]])
    A = _linear_actor(mu[0], l[0])
    _, _, _, head = sac.policy_forward(A, np.zeros((1, 2)), eps, cfg)
    g = sac.policy_head_backward(head, np.ones((1, 2)), np.array([0.7]), cfg)
    tl = torch.tensor(l, requires_grad=True)
    lc = torch.clamp(tl, -20.0, 2.0)
    u = torch.tensor(mu) + torch.exp(lc) * torch.tensor(eps)
    a = torch.tanh(u)
    lp = (-0.5 * torch.tensor(eps) ** 2 - lc - 0.5 * np.log(2 * np.pi)
          - 2 * (np.log(2.0) - u - torch.nn.functional.softplus(-2 * u))).sum()
    (a.sum() + 0.7 * lp).backward()
    assert np.allclose(g[0, 2:], tl.grad.numpy()[0], rtol=1e-12, atol=1e-14)
    assert np.all(g[0, 2:] != 0.0)


# ----------------------------------------------------------------------------- whole-step gradients

def _torch_mlp(params, x, relu_last=False):
    a = x
    for l, (W, b) in enumerate(params):
        a = torch.nn.functional.linear(a, W, b)
        if l < len(params) - 1:
            a = torch.relu(a)
    return a


def _tp(flat, shapes, grad):
    return [(torch.tensor(W, requires_grad=grad), torch.tensor(b, requires_grad=grad))
            for W, b in mlp.unflatten(flat, shapes)]


def test_sac_grads_match_torch_autograd():
    cfg, r, st = small_problem("sac")
    B = 48
    idx, batch = r.sample(B, 6126, 0)
    eps, eps2 = sac.draw_noise(6126, 0, B, cfg.act_dim)
    grads, sums = sac.sac_grads(st, batch, eps, eps2, cfg, B)

    ash, csh = sac.actor_shapes(cfg), sac.critic_shapes(cfg)
    s, a, rr, s2, d = [torch.tensor(np.asarray(batch[k], np.float64)) for k in ("obs", "act", "rew", "next_obs", "done")]
    A = _tp(st.actor, ash, True)
    Q1, Q2 = _tp(st.q1, csh, True), _tp(st.q2, csh, True)
    Q1t, Q2t = _tp(st.q1_targ, csh, False), _tp(st.q2_targ, csh, False)
    log_alpha = torch.tensor(st.log_alpha, dtype=torch.float64, requires_grad=True)
    m = cfg.act_dim

    def pol(x, e):
        H = _torch_mlp(A, x)
        mu, l = H[:, :m], H[:, m:]
        lc = torch.clamp(l, cfg.log_std_min, cfg.log_std_max)
        u = mu + torch.exp(lc) * e
        lp = (-0.5 * e ** 2 - lc - 0.5 * np.log(2 * np.pi)
              - 2 * (np.log(2.0) - u - torch.nn.functional.softplus(-2 * u))).sum(1)
        return torch.tanh(u), lp

    alpha = torch.exp(log_alpha).detach()
    with torch.no_grad():
        a2, lp2 = pol(s2, torch.tensor(eps2))
        y = rr + cfg.gamma * (1 - d) * (torch.minimum(_torch_mlp(Q1t, torch.cat([s2, a2], 1))[:, 0],
                                                      _torch_mlp(Q2t, torch.cat([s2, a2], 1))[:, 0]) - alpha * lp2)
    LQ = ((_torch_mlp(Q1, torch.cat([s, a], 1))[:, 0] - y) ** 2 + (_torch_mlp(Q2, torch.cat([s, a], 1))[:, 0] - y) ** 2).mean()
    at, lpt = pol(s, torch.tensor(eps))
    Q1d = [(W.detach(), b.detach()) for W, b in Q1]
    Q2d = [(W.detach(), b.detach()) for W, b in Q2]
    Lpi = (alpha * lpt - torch.minimum(_torch_mlp(Q1d, torch.cat([s, at], 1))[:, 0],
                                       _torch_mlp(Q2d, torch.cat([s, at], 1))[:, 0])).mean()
    La = -(log_alpha * (lpt.detach() + cfg.target_entropy)).mean()
    (LQ + Lpi + La).backward()
    flat = lambda P: np.concatenate([np.concatenate([W.grad.numpy().ravel(), b.grad.numpy()]) for W, b in P])
    assert np.allclose(grads["q1"], flat(Q1), rtol=1e-10, atol=1e-13)
    assert np.allclose(grads["q2"], flat(Q2), rtol=1e-10, atol=1e-13)
    assert np.allclose(grads["actor"], flat(A), rtol=1e-10, atol=1e-13)
    assert np.allclose(grads["log_alpha"][0], log_alpha.grad.item(), rtol=1e-12)
    assert np.isclose(sums["lq"] / B, LQ.item(), rtol=1e-12)
    assert np.isclose(sums["lpi"] / B, Lpi.item(), rtol=1e-12)


def test_td3_grads_match_torch_autograd():
    cfg, r, st = small_problem("td3")
    B = 40
    k = 1  # delayed step
    assert td3.is_delayed(k, cfg)
    idx, batch = r.sample(B, 6126, k)
    xi = td3.draw_smoothing(6126, k, B, cfg)
    grads, sums = td3.td3_grads(st, batch, xi, cfg, B, k)
    ash, csh = sac.actor_shapes(cfg, td3=True), sac.critic_shapes(cfg)
    s, a, rr, s2, d = [torch.tensor(np.asarray(batch[kk], np.float64)) for kk in ("obs", "act", "rew", "next_obs", "done")]
    A = _tp(st.actor, ash, True)
    At = _tp(st.actor_targ, ash, False)
    Q1, Q2 = _tp(st.q1, csh, True), _tp(st.q2, csh, True)
    Q1t, Q2t = _tp(st.q1_targ, csh, False), _tp(st.q2_targ, csh, False)
    with torch.no_grad():
        a2 = torch.clamp(torch.tanh(_torch_mlp(At, s2)) + torch.tensor(xi), -1, 1)
        y = rr + cfg.gamma * (1 - d) * torch.minimum(_torch_mlp(Q1t, torch.cat([s2, a2], 1))[:, 0],
                                                     _torch_mlp(Q2t, torch.cat([s2, a2], 1))[:, 0])
    LQ = ((_torch_mlp(Q1, torch.cat([s, a], 1))[:, 0] - y) ** 2 + (_torch_mlp(Q2, torch.cat([s, a], 1))[:, 0] - y) ** 2).mean()
    Q1d = [(W.detach(), b.detach()) for W, b in Q1]
    Lpi = -_torch_mlp(Q1d, torch.cat([s, torch.tanh(_torch_mlp(A, s))], 1))[:, 0].mean()
    (LQ + Lpi).backward()
    flat = lambda P: np.concatenate([np.concatenate([W.grad.numpy().ravel(), b.grad.numpy()]) for W, b in P])
    assert np.allclose(grads["q1"], flat(Q1), rtol=1e-10, atol=1e-13)
    assert np.allclose(grads["q2"], flat(Q2), rtol=1e-10, atol=1e-13)
    assert np.allclose(grads["actor"], flat(A), rtol=1e-10, atol=1e-13)


def test_td3_non_delayed_step_keeps_actor_and_targets():
    cfg, r, st = small_problem("td3")
    st1, stats, _ = td3.td3_step(st, r, 32, 6126, cfg)  # k = 0: not delayed
    assert np.array_equal(st1.actor, st.actor) and np.array_equal(st1.actor_targ, st.actor_targ)
    assert np.array_equal(st1.q1_targ, st.q1_targ) and st1.opt["actor"].t == 0 and st1.opt["q1"].t == 1
    st2, _, _ = td3.td3_step(st1, r, 32, 6126, cfg)  # k = 1: delayed
    assert not np.array_equal(st2.actor, st1.actor) and st2.opt["actor"].t == 1
    assert np.allclose(st2.q1_targ, cfg.tau * st2.q1 + (1 - cfg.tau) * st1.q1_targ, rtol=0, atol=1e-15)


# ----------------------------------------------------------------------------- special cases

def test_bellman_target_special_cases():
    cfg, r, st = small_problem("sac")
    B = 32
    idx, batch = r.sample(B, 6126, 0)
    eps, eps2 = sac.draw_noise(6126, 0, B, cfg.act_dim)
    # gamma = 0 and alpha = 0 -> y = r exactly
    cfg0 = sac.Config(obs_dim=cfg.obs_dim, act_dim=cfg.act_dim, hidden=cfg.hidden, n_hidden=cfg.n_hidden, gamma=0.0)
    st0 = st.copy()
    st0.log_alpha = -1000.0
    _, sums = sac.sac_grads(st0, batch, eps, eps2, cfg0, B, actor=False)
    assert np.array_equal(sums["y"], np.asarray(batch["rew"], np.float64))
    # d = 1 drops the bootstrap whatever gamma and alpha
    b1 = dict(batch)
    b1["done"] = np.ones(B, np.float32)
    _, sums = sac.sac_grads(st, b1, eps, eps2, cfg, B, actor=False)
    assert np.array_equal(sums["y"], np.asarray(batch["rew"], np.float64))


def test_alpha_gradient_vs_finite_difference():
    cfg, r, st = small_problem("sac")
    B = 32
    idx, batch = r.sample(B, 6126, 0)
    eps, eps2 = sac.draw_noise(6126, 0, B, cfg.act_dim)
    g, sums = sac.sac_grads(st, batch, eps, eps2, cfg, B)
    logp_mean = sums["logp"] / B
    La = lambda la: -la * (logp_mean + cfg.target_entropy)  # log pi~ detached
    h = 1e-6
    fd = (La(st.log_alpha + h) - La(st.log_alpha - h)) / (2 * h)
    assert abs(fd - g["log_alpha"][0]) < 1e-8


def test_critic_fixed_point_toy():
    # 1-state 1-action toy, s2 = s, d = 0, alpha = 0 -> Q -> r / (1 - gamma) within 1e-2.
    # The actor is frozen at a deterministic action equal to the stored one (mu = atanh(a), log std = -20).
    o, m = 2, 1
    gamma, rew, act = 0.8, 1.0, 0.25
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=8, n_hidden=1, gamma=gamma, tau=0.1,
                     lr_critic=5e-3, lr_actor=0.0, alpha_auto=False)
    ring = oring.Ring(o, m, 4)
    s = np.array([[0.5, -0.3]], np.float32)
    ring.push(obs=s, act=np.array([[act]], np.float32), rew=np.array([rew], np.float32),
              next_obs=s, done=np.zeros(1, np.float32))
    ash = sac.actor_shapes(cfg)
    actor = mlp.flatten([(np.zeros((8, o)), np.zeros(8)),
                         (np.zeros((2, 8)), np.array([np.arctanh(act), -20.0]))])
    p = synthdata.init_params(o, m, 8, 1, seed=3)
    st = sac.State.create(actor, p["q1"], p["q2"], log_alpha=-1000.0)
    for k in range(3000):
        st, stats, _ = sac.sac_step(st, ring, 1, 6126, cfg)
    q_star = rew / (1 - gamma)
    assert abs(stats["q1_mean"] - q_star) < 1e-2 and abs(stats["q2_mean"] - q_star) < 1e-2


def test_determinism_bit_identical():
    cfg, r, st = small_problem("sac")
    a, b = st.copy(), st.copy()
    for _ in range(3):
        a, sa, _ = sac.sac_step(a, r, 32, 6126, cfg)
        b, sb, _ = sac.sac_step(b, r, 32, 6126, cfg)
    assert np.array_equal(a.actor, b.actor) and np.array_equal(a.q1, b.q1) and sa == sb


def test_min_tie_split_half():
    w1, w2 = sac.min_weights(np.array([1.0, 2.0, 3.0]), np.array([2.0, 1.0, 3.0]))
    assert np.array_equal(w1, [1.0, 0.0, 0.5]) and np.array_equal(w2, [0.0, 1.0, 0.5])
    # torch.minimum splits the gradient 1/2-1/2 on a tie
    x = torch.tensor([3.0], dtype=torch.float64, requires_grad=True)
    yv = torch.tensor([3.0], dtype=torch.float64, requires_grad=True)
    torch.minimum(x, yv).sum().backward()
    assert x.grad.item() == 0.5 and yv.grad.item() == 0.5


# ----------------------------------------------------------------------------- behavioural pins (signs of every loss term)

def _const_critic(o, m, h, b_out):
    """All-zero hidden weights: Z = 0, ReLU'(0) = 0, so the net stays the constant b_out forever."""
    return mlp.flatten([(np.zeros((h, o + m)), np.zeros(h)), (np.zeros((1, h)), np.array([b_out]))])


def _one_transition_ring(o, m, rew=1.0, act=0.1, copies=1024):
    """One state-action pair stored ``copies`` times (fill >= B)."""
    ring = oring.Ring(o, m, copies)
    s = np.full((copies, o), 0.3, np.float32)
    ring.push(obs=s, act=np.full((copies, m), act, np.float32), rew=np.full(copies, rew, np.float32),
              next_obs=s, done=np.zeros(copies, np.float32))
    return ring


def test_soft_bellman_fixed_point_entropy_term():
    """Constant critic b, frozen policy with known E[log pi]: b* = (r - gamma alpha E[log pi]) / (1 - gamma).

    E[log pi] under the sampling law u ~ N(mu, sigma) is evaluated by Gauss-Hermite quadrature;
    a dropped or sign-flipped entropy term moves b* by ~0.5 here."""
    o, m, h = 2, 1, 4
    mu, l = 0.3, -0.4
    gamma, alpha, rew = 0.5, 0.5, 1.0
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=1, gamma=gamma, tau=1.0,
                     lr_critic=1e-2, lr_actor=0.0, alpha_auto=False)
    actor = mlp.flatten([(np.zeros((h, o)), np.zeros(h)), (np.zeros((2, h)), np.array([mu, l]))])
    st = sac.State.create(actor, _const_critic(o, m, h, 0.0), _const_critic(o, m, h, 0.0), log_alpha=np.log(alpha))
    ring = _one_transition_ring(o, m, rew)
    bs = []
    for k in range(1500):
        st, stats, _ = sac.sac_step(st, ring, 1024, 6126, cfg)
        bs.append(stats["q1_mean"])
    x, w = np.polynomial.hermite_e.hermegauss(80)  # E_{z~N(0,1)} f(z) = sum w f(x) / sqrt(2 pi)
    sigma = np.exp(l)
    A = mlp.unflatten(actor, sac.actor_shapes(cfg))
    _, lp, _, _ = sac.policy_forward(A, np.zeros((x.size, o)), x.reshape(-1, 1), cfg)
    e_logp = np.sum(w * lp) / np.sqrt(2 * np.pi)
    b_star = (rew - gamma * alpha * e_logp) / (1 - gamma)
    assert abs(np.mean(bs[-300:]) - b_star) < 2e-2, (np.mean(bs[-300:]), b_star)


def test_actor_climbs_critic_and_entropy():
    o, m, h = 2, 1, 4
    # (a) increasing critic Q = a + 10 (one hidden unit on the action column), alpha ~ 0 -> mean action rises
    W1 = np.zeros((1, o + m))
    W1[0, o] = 1.0
    q = mlp.flatten([(W1, np.array([10.0])), (np.ones((1, 1)), np.zeros(1))])
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=1, n_hidden=1, lr_critic=0.0, lr_actor=1e-2, alpha_auto=False)
    actor = mlp.flatten([(np.zeros((1, o)), np.zeros(1)), (np.zeros((2, 1)), np.array([0.0, -1.0]))])
    st = sac.State.create(actor, q, q, log_alpha=-20.0)
    ring = _one_transition_ring(o, m)
    _, s0, _ = sac.sac_step(st, ring, 256, 1, cfg)
    for _ in range(50):
        st, stats, _ = sac.sac_step(st, ring, 256, 1, cfg)
    mu_final = st.actor[-2]
    assert mu_final > 0.3, mu_final
    # (b) flat critic, alpha = 1: maximum entropy -> log sigma grows, mean log pi falls
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=1, lr_critic=0.0, lr_actor=1e-2, alpha_auto=False)
    actor = mlp.flatten([(np.zeros((h, o)), np.zeros(h)), (np.zeros((2, h)), np.array([0.0, -2.0]))])
    st = sac.State.create(actor, _const_critic(o, m, h, 0.0), _const_critic(o, m, h, 0.0), log_alpha=0.0)
    _, s0, _ = sac.sac_step(st, ring, 256, 1, cfg)
    for _ in range(50):
        st, stats, _ = sac.sac_step(st, ring, 256, 1, cfg)
    assert st.actor[-1] > -2.0 + 0.3 and stats["logp_mean"] < s0["logp_mean"] - 0.2


def test_temperature_moves_toward_target_entropy():
    # L_alpha = -log alpha (log pi + H_bar): if the policy entropy is above target (log pi + H_bar < 0), alpha falls
    o, m, h = 2, 1, 4
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=1, lr_critic=0.0, lr_actor=0.0, lr_alpha=1e-2,
                     target_entropy=-4.0)
    actor = mlp.flatten([(np.zeros((h, o)), np.zeros(h)), (np.zeros((2, h)), np.array([0.0, 0.0]))])
    st = sac.State.create(actor, _const_critic(o, m, h, 0.0), _const_critic(o, m, h, 0.0), log_alpha=0.0)
    ring = _one_transition_ring(o, m)
    for _ in range(20):
        st, stats, _ = sac.sac_step(st, ring, 256, 1, cfg)
    assert st.log_alpha < -0.15


# ----------------------------------------------------------------------------- DDPG (f4)

def test_ddpg_grads_match_torch_autograd():
    from oracle import ddpg
    cfg, r, st = small_problem("td3")
    B = 40
    idx, batch = r.sample(B, 6126, 0)
    grads, sums = ddpg.ddpg_grads(st, batch, cfg, B)
    ash, csh = sac.actor_shapes(cfg, td3=True), sac.critic_shapes(cfg)
    s, a, rr, s2, d = [torch.tensor(np.asarray(batch[kk], np.float64)) for kk in ("obs", "act", "rew", "next_obs", "done")]
    A = _tp(st.actor, ash, True)
    At = _tp(st.actor_targ, ash, False)
    Q1 = _tp(st.q1, csh, True)
    Q1t = _tp(st.q1_targ, csh, False)
    with torch.no_grad():
        y = rr + cfg.gamma * (1 - d) * _torch_mlp(Q1t, torch.cat([s2, torch.tanh(_torch_mlp(At, s2))], 1))[:, 0]
    LQ = ((_torch_mlp(Q1, torch.cat([s, a], 1))[:, 0] - y) ** 2).mean()
    Q1d = [(W.detach(), b.detach()) for W, b in Q1]
    Lpi = -_torch_mlp(Q1d, torch.cat([s, torch.tanh(_torch_mlp(A, s))], 1))[:, 0].mean()
    (LQ + Lpi).backward()
    flat = lambda P: np.concatenate([np.concatenate([W.grad.numpy().ravel(), b.grad.numpy()]) for W, b in P])
    assert np.allclose(grads["q1"], flat(Q1), rtol=1e-10, atol=1e-13)
    assert np.allclose(grads["actor"], flat(A), rtol=1e-10, atol=1e-13)
    assert np.isclose(sums["lq"] / B, LQ.item(), rtol=1e-12) and np.isclose(sums["lpi"] / B, Lpi.item(), rtol=1e-12)


def test_ddpg_equals_td3_with_tied_twins_no_delay_no_noise():
    """DDPG is TD3 with policy delay 1, no target smoothing and the twin critic tied to the first: with
    Q2 = Q1 (and Q2' = Q1') the twins receive identical updates, min(Q1', Q2') = Q1', and TD3's critic
    loss is twice DDPG's.  (The GPU path runs DDPG exactly this way.)"""
    from oracle import ddpg
    cfg, r, st = small_problem("td3")
    cfg.td3_policy_delay, cfg.td3_noise, cfg.td3_noise_clip = 1, 0.0, 0.0
    st_t = sac.State.create(st.actor, st.q1, st.q1, log_alpha=0.0, actor_targ=st.actor)
    st_d = st_t.copy()
    for _ in range(4):
        st_t, s_t, _ = td3.td3_step(st_t, r, 48, 6126, cfg)
        st_d, s_d, _ = ddpg.ddpg_step(st_d, r, 48, 6126, cfg)
        assert np.isclose(s_t["critic_loss"], 2 * s_d["critic_loss"], rtol=1e-12)
        assert np.isclose(s_t["actor_loss"], s_d["actor_loss"], rtol=1e-12)
    for n in ("actor", "q1", "q1_targ", "actor_targ"):
        assert np.allclose(getattr(st_t, n), getattr(st_d, n), rtol=0, atol=1e-14), n
    assert np.array_equal(st_t.q1, st_t.q2)
