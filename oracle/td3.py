"""One TD3 update step in float64, Jacobi order (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:576 ("our framework can also be easily extended to ... TD3",
citing Fujimoto et al. 2018).  Readings #18 and #3: policy delay 2,
target smoothing noise 0.2 clipped to 0.5, deterministic tanh actor, Q1-only
actor loss, targets (including the target actor) Polyak-averaged only on
delayed steps, all losses evaluated at step-k parameters (Jacobi).  Step k:

 1. indices and gather as in SAC;
 2. xi = clip(0.2 n, -0.5, 0.5), n ~ N(0,1) from stream S_SMOOTH;
 3. a' = clip(tanh(MLP_phi'(s2)) + xi, -1, 1);
 4. y = r + gamma (1-d) min(Q'_1, Q'_2)(s2, a');
 5. L_Q as in SAC, Adam on the critics (every step);
 6. if (k+1) mod delay == 0: L_pi = -(1/B) sum_j Q_1,k(s_j, tanh(MLP_phi(s_j))),
    Adam on phi, Polyak on theta'_1, theta'_2 and phi'.
"""

import numpy as np

from . import mlp, optim, philox
from .sac import actor_shapes, critic_shapes, critic_q, _batch_f64


def is_delayed(step, cfg):
    return (step + 1) % cfg.td3_policy_delay == 0


def td3_grads(st, batch, xi, cfg, B_global, step, critic=True, actor=True, decisions=None):
    """decisions: as sac.sac_grads ("q1", "q2", "q1_pi", "actor" ReLU masks; reading #25)."""
    dec = decisions or {}
    s, a, r, s2, d = _batch_f64(batch)
    o, m = cfg.obs_dim, cfg.act_dim
    ash = actor_shapes(cfg, td3=True)
    cs = critic_shapes(cfg)
    grads, sums = {}, {}
    if critic:
        At = mlp.unflatten(st.actor_targ, ash)
        z2, _ = mlp.forward(At, s2)
        a2 = np.clip(np.tanh(z2) + xi, -1.0, 1.0)
        qt1, _ = critic_q(mlp.unflatten(st.q1_targ, cs), s2, a2)
        qt2, _ = critic_q(mlp.unflatten(st.q2_targ, cs), s2, a2)
        y = r + cfg.gamma * (1.0 - d) * np.minimum(qt1, qt2)
        lq = 0.0
        for i, th in enumerate((st.q1, st.q2)):
            P = mlp.unflatten(th, cs)
            q, cache = critic_q(P, s, a, dec.get(f"q{i + 1}"))
            g, _ = mlp.backward(P, cache, (2.0 * (q - y) / B_global).reshape(-1, 1))
            grads[f"q{i + 1}"] = mlp.flatten(g)
            lq = lq + np.sum((q - y) ** 2)
            sums[f"q{i + 1}"] = np.sum(q)
            sums[f"q{i + 1}_abs"] = np.sum(np.abs(q))  # conditioning of the mean (test tolerance scale)
        sums["lq"] = lq
        sums["y"] = y
    if actor and is_delayed(step, cfg):
        A = mlp.unflatten(st.actor, ash)
        z, acache = mlp.forward(A, s, dec.get("actor"))
        at = np.tanh(z)
        Q1 = mlp.unflatten(st.q1, cs)
        q, cache = critic_q(Q1, s, at, dec.get("q1_pi"))
        _, dX = mlp.backward(Q1, cache, np.full((s.shape[0], 1), -1.0 / B_global))
        g_a = dX[:, o:o + m]
        dZ = g_a * (1.0 - at * at)
        g, _ = mlp.backward(A, acache, dZ)
        grads["actor"] = mlp.flatten(g)
        sums["lpi"] = -np.sum(q)
        sums["lpi_abs"] = np.sum(np.abs(q))  # conditioning of the mean (test tolerance scale)
    return grads, sums


def td3_apply(st, grads, cfg, step, critic=True, actor=True):
    st = st.copy()
    adam = lambda th, g, key, lr: optim.adam_step(th, g, st.opt[key], lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
    delayed = is_delayed(step, cfg)
    if critic:
        st.q1 = adam(st.q1, grads["q1"], "q1", cfg.lr_critic)
        st.q2 = adam(st.q2, grads["q2"], "q2", cfg.lr_critic)
    if actor and delayed:
        st.actor = adam(st.actor, grads["actor"], "actor", cfg.lr_actor)
    if delayed:
        if critic:
            st.q1_targ = optim.polyak(st.q1_targ, st.q1, cfg.tau)
            st.q2_targ = optim.polyak(st.q2_targ, st.q2, cfg.tau)
        if actor:
            st.actor_targ = optim.polyak(st.actor_targ, st.actor, cfg.tau)
    st.step += 1
    return st


def draw_smoothing(seed, step, batch, cfg, row0=0):
    n = philox.normals(seed, step, philox.S_SMOOTH, batch, cfg.act_dim, row0=row0)
    return np.clip(cfg.td3_noise * n, -cfg.td3_noise_clip, cfg.td3_noise_clip)


def stats_of(st, sums, B):
    return dict(step=st.step, critic_loss=float(sums["lq"] / B),
                actor_loss=float(sums.get("lpi", 0.0) / B), actor_loss_abs=float(sums.get("lpi_abs", 0.0) / B), alpha=0.0, alpha_loss=0.0,
                q1_mean=float(sums["q1"] / B), q2_mean=float(sums["q2"] / B), logp_mean=0.0,
                q1_mean_abs=float(sums.get("q1_abs", 0.0) / B), q2_mean_abs=float(sums.get("q2_abs", 0.0) / B))


def td3_step(st, ring, B, seed, cfg):
    k = st.step
    idx, batch = ring.sample(B, seed, k)
    xi = draw_smoothing(seed, k, B, cfg)
    grads, sums = td3_grads(st, batch, xi, cfg, B, k)
    stats = stats_of(st, sums, B)
    return td3_apply(st, grads, cfg, k), stats, idx
