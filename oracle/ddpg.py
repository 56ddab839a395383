"""One DDPG update step in float64, Jacobi order (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md §8(f) f4: DDPG is one of the off-policy actor-critics the paper names (its comparison
systems run APE-DDPG) and the deterministic-policy ancestor of TD3.  Lillicrap et al.'s
update, in the same Jacobi order and conventions as oracle/td3.py (readings #3, #10, #11; DESIGN.md reading
#23): one critic Q with target Q', deterministic tanh actor with target actor, no target smoothing, no
policy delay.  Step k:

 1. indices and gather as in SAC;
 2. a' = tanh(MLP_phi'(s2));  y = r + gamma (1-d) Q'(s2, a'), a constant;
 3. L_Q = (1/B) sum_j (Q(s_j, a_j) - y_j)^2;          Adam on theta;
 4. L_pi = -(1/B) sum_j Q_k(s_j, tanh(MLP_phi(s_j)))   (critic at step k);  Adam on phi;
 5. Polyak theta' <- tau theta_new + (1 - tau) theta',  phi' <- tau phi_new + (1 - tau) phi'.
"""

import numpy as np

from . import mlp, optim
from .sac import actor_shapes, critic_shapes, critic_q, _batch_f64


def ddpg_grads(st, batch, cfg, B_global):
    s, a, r, s2, d = _batch_f64(batch)
    o, m = cfg.obs_dim, cfg.act_dim
    ash, cs = actor_shapes(cfg, td3=True), critic_shapes(cfg)
    At = mlp.unflatten(st.actor_targ, ash)
    z2, _ = mlp.forward(At, s2)
    qt, _ = critic_q(mlp.unflatten(st.q1_targ, cs), s2, np.tanh(z2))
    y = r + cfg.gamma * (1.0 - d) * qt
    Q = mlp.unflatten(st.q1, cs)
    q, cache = critic_q(Q, s, a)
    gq, _ = mlp.backward(Q, cache, (2.0 * (q - y) / B_global).reshape(-1, 1))
    A = mlp.unflatten(st.actor, ash)
    z, acache = mlp.forward(A, s)
    at = np.tanh(z)
    qa, ccache = critic_q(Q, s, at)
    _, dX = mlp.backward(Q, ccache, np.full((s.shape[0], 1), -1.0 / B_global))
    ga, _ = mlp.backward(A, acache, dX[:, o:o + m] * (1.0 - at * at))
    grads = {"q1": mlp.flatten(gq), "actor": mlp.flatten(ga)}
    sums = {"lq": np.sum((q - y) ** 2), "q1": np.sum(q), "q1_abs": np.sum(np.abs(q)), "lpi": -np.sum(qa),
            "lpi_abs": np.sum(np.abs(qa)), "y": y}
    return grads, sums


def ddpg_apply(st, grads, cfg):
    st = st.copy()
    st.q1 = optim.adam_step(st.q1, grads["q1"], st.opt["q1"], cfg.lr_critic, cfg.beta1, cfg.beta2, cfg.adam_eps)
    st.actor = optim.adam_step(st.actor, grads["actor"], st.opt["actor"], cfg.lr_actor, cfg.beta1, cfg.beta2,
                               cfg.adam_eps)
    st.q1_targ = optim.polyak(st.q1_targ, st.q1, cfg.tau)
    st.actor_targ = optim.polyak(st.actor_targ, st.actor, cfg.tau)
    st.step += 1
    return st


def stats_of(st, sums, B):
    return dict(step=st.step, critic_loss=float(sums["lq"] / B), actor_loss=float(sums["lpi"] / B),
                actor_loss_abs=float(sums["lpi_abs"] / B), alpha=0.0, alpha_loss=0.0,
                q1_mean=float(sums["q1"] / B), q1_mean_abs=float(sums["q1_abs"] / B), logp_mean=0.0)


def ddpg_step(st, ring, B, seed, cfg):
    """State fields used: actor, actor_targ, q1, q1_targ (q2 / q2_targ are ignored)."""
    k = st.step
    idx, batch = ring.sample(B, seed, k)
    grads, sums = ddpg_grads(st, batch, cfg, B)
    stats = stats_of(st, sums, B)
    return ddpg_apply(st, grads, cfg), stats, idx
