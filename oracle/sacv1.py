"""One SAC v1 update step (state-value network) in float64, Jacobi order (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md §8(f) f4: the original soft actor-critic the paper cites (haarnoja2018soft), which keeps
a state-value network V_psi with a Polyak target V_psibar next to the twin soft Q-functions and the
squashed-Gaussian policy.  Written in the conventions of oracle/sac.py (readings #3, #6, #9, #10, #11) and
DESIGN.md reading #24 (the v1 losses as mean squared errors, no 1/2, like L_Q; the temperature handled as
in SAC, learned only if alpha_auto).  Step k, every loss at the step-k parameters:

 1. indices and gather as in SAC; eps = the S_EPS normals of the s rows (no a' is drawn: v1 has no
    next-state action);
 2. a~, log pi~ = pi_phi(s; eps);
 3. y_V = min(Q1(s, a~), Q2(s, a~)) - alpha log pi~            (a constant)
    L_V = (1/B) sum_j (V(s_j) - y_V,j)^2;
 4. y_Q = r + gamma (1 - d) V_psibar(s2)                        (a constant)
    L_Q = (1/B) sum_j sum_i (Q_i(s_j, a_j) - y_Q,j)^2;
 5. L_pi = (1/B) sum_j (alpha log pi~_j - min_i Q_i(s_j, a~_j))  (SAC's policy loss, reading #9 on ties);
    L_alpha as SAC;
 6. Adam on theta_1, theta_2, psi (lr_critic), phi (lr_actor), log alpha (if auto); Polyak
    psibar <- tau psi_new + (1 - tau) psibar.  There are no target Q networks.
"""

from dataclasses import dataclass, field

import numpy as np

from . import mlp, optim, philox
from .sac import actor_shapes, critic_shapes, critic_q, min_weights, policy_forward, policy_head_backward, _batch_f64


def value_shapes(cfg):
    return mlp.layer_dims(cfg.obs_dim, cfg.hidden, cfg.n_hidden, 1)


@dataclass
class State:
    actor: np.ndarray
    q1: np.ndarray
    q2: np.ndarray
    v: np.ndarray
    v_targ: np.ndarray
    log_alpha: float
    opt: dict = field(default_factory=dict)
    step: int = 0

    @staticmethod
    def create(actor, q1, q2, v, v_targ=None, log_alpha=0.0):
        f = lambda x: np.asarray(x, dtype=np.float64).copy()
        st = State(actor=f(actor), q1=f(q1), q2=f(q2), v=f(v), v_targ=f(v if v_targ is None else v_targ),
                   log_alpha=float(log_alpha))
        st.opt = {k: optim.AdamState(getattr(st, k).size) for k in ("actor", "q1", "q2", "v")}
        st.opt["alpha"] = optim.AdamState(1)
        return st

    def copy(self):
        c = State(actor=self.actor.copy(), q1=self.q1.copy(), q2=self.q2.copy(), v=self.v.copy(),
                  v_targ=self.v_targ.copy(), log_alpha=self.log_alpha, step=self.step)
        c.opt = {k: o.copy() for k, o in self.opt.items()}
        return c


def value_of(params, s):
    v, cache = mlp.forward(params, s)
    return v[:, 0], cache


def sacv1_grads(st, batch, eps, cfg, B_global):
    s, a, r, s2, d = _batch_f64(batch)
    m, o = cfg.act_dim, cfg.obs_dim
    alpha = np.exp(st.log_alpha)
    A = mlp.unflatten(st.actor, actor_shapes(cfg))
    cs, vs = critic_shapes(cfg), value_shapes(cfg)
    Q = [mlp.unflatten(st.q1, cs), mlp.unflatten(st.q2, cs)]
    V = mlp.unflatten(st.v, vs)
    grads, sums = {}, {}
    # 2. the policy on s
    at, logpt, acache, head = policy_forward(A, s, eps, cfg)
    qa, qcaches = [], []
    for i in range(2):
        q, cache = critic_q(Q[i], s, at)
        qa.append(q)
        qcaches.append(cache)
    qmin = np.minimum(qa[0], qa[1])
    # 3. value loss
    y_v = qmin - alpha * logpt
    v, vcache = value_of(V, s)
    gv, _ = mlp.backward(V, vcache, (2.0 * (v - y_v) / B_global).reshape(-1, 1))
    grads["v"] = mlp.flatten(gv)
    sums["lv"] = np.sum((v - y_v) ** 2)
    sums["v"] = np.sum(v)
    sums["y_v"] = y_v
    # 4. soft Q losses against the target value of the next state
    vt, _ = value_of(mlp.unflatten(st.v_targ, vs), s2)
    y = r + cfg.gamma * (1.0 - d) * vt
    lq = 0.0
    for i in range(2):
        q, cache = critic_q(Q[i], s, a)
        g, _ = mlp.backward(Q[i], cache, (2.0 * (q - y) / B_global).reshape(-1, 1))
        grads[f"q{i + 1}"] = mlp.flatten(g)
        lq = lq + np.sum((q - y) ** 2)
        sums[f"q{i + 1}"] = np.sum(q)
        sums[f"q{i + 1}_abs"] = np.sum(np.abs(q))
    sums["lq"] = lq
    sums["y"] = y
    # 5. policy loss through the critics (step-k theta), then the temperature
    w1, w2 = min_weights(qa[0], qa[1])
    g_a = np.zeros_like(at)
    for i, w in enumerate((w1, w2)):
        _, dX = mlp.backward(Q[i], qcaches[i], (-w / B_global).reshape(-1, 1))
        g_a += dX[:, o:o + m]
    dH = policy_head_backward(head, g_a, np.full(s.shape[0], alpha / B_global), cfg)
    g, _ = mlp.backward(A, acache, dH)
    grads["actor"] = mlp.flatten(g)
    if cfg.alpha_auto:
        grads["log_alpha"] = np.array([-np.sum(logpt + cfg.target_entropy) / B_global])
    sums["lpi"] = np.sum(alpha * logpt - qmin)
    sums["lpi_abs"] = np.sum(np.abs(alpha * logpt - qmin))
    sums["logp"] = np.sum(logpt)
    return grads, sums


def sacv1_apply(st, grads, cfg):
    st = st.copy()
    adam = lambda th, g, key, lr: optim.adam_step(th, g, st.opt[key], lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
    st.q1 = adam(st.q1, grads["q1"], "q1", cfg.lr_critic)
    st.q2 = adam(st.q2, grads["q2"], "q2", cfg.lr_critic)
    st.v = adam(st.v, grads["v"], "v", cfg.lr_critic)
    st.v_targ = optim.polyak(st.v_targ, st.v, cfg.tau)
    st.actor = adam(st.actor, grads["actor"], "actor", cfg.lr_actor)
    if cfg.alpha_auto:
        st.log_alpha = float(adam(np.array([st.log_alpha]), grads["log_alpha"], "alpha", cfg.lr_alpha)[0])
    st.step += 1
    return st


def stats_of(st, sums, B, cfg):
    alpha = float(np.exp(st.log_alpha))
    return dict(step=st.step, critic_loss=float(sums["lq"] / B), value_loss=float(sums["lv"] / B),
                actor_loss=float(sums["lpi"] / B), actor_loss_abs=float(sums["lpi_abs"] / B), alpha=alpha,
                alpha_loss=float(-st.log_alpha * (sums["logp"] / B + cfg.target_entropy)),
                q1_mean=float(sums["q1"] / B), q2_mean=float(sums["q2"] / B),
                q1_mean_abs=float(sums["q1_abs"] / B), q2_mean_abs=float(sums["q2_abs"] / B),
                logp_mean=float(sums["logp"] / B))


def sacv1_step(st, ring, B, seed, cfg):
    """One full single-device SAC v1 update at step k = st.step.  Returns (state', stats, idx)."""
    k = st.step
    idx, batch = ring.sample(B, seed, k)
    eps = philox.normals(seed, k, philox.S_EPS, B, cfg.act_dim)
    grads, sums = sacv1_grads(st, batch, eps, cfg, B)
    stats = stats_of(st, sums, B, cfg)
    return sacv1_apply(st, grads, cfg), stats, idx
