"""One SAC update step in float64, Jacobi order (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md §3.2.2 (SAC, double-Q "two value networks Q1 and
Q2", "updated ... together with the target network"), SPEC S:368 (losses) and
north_star (soft Bellman target from the target networks, temperature
gradient), in the step order of SURVEY.md §8(c) "SAC step k":

 1. indices idx_j (philox.sample_indices) and the gathered (s, a, r, s2, d);
 2. noise eps (stream S_EPS, for the action on s) and eps' (S_EPS2, on s2);
 3. squashed-Gaussian policy: [mu | l] = MLP_phi(s); lc = clamp(l, lo, hi);
    sigma = exp(lc); u = mu + sigma*eps; a = tanh(u);
    log pi = sum_i [-eps_i^2/2 - lc_i - ln(2 pi)/2 - 2(ln 2 - u_i - softplus(-2 u_i))];
 4. y = r + gamma (1-d) (min(Q'_1, Q'_2)(s2, a') - alpha_k log pi'), a constant;
 5. L_Q = (1/B) sum_j [(Q_1(s,a) - y)^2 + (Q_2(s,a) - y)^2];
 6. L_pi = (1/B) sum_j [alpha_k log pi~ - min(Q_1, Q_2)(s, a~)], gradient through
    a~ and log pi~, critics held at theta_k (Jacobi, reading #3), min tie split 1/2-1/2;
 7. g_log_alpha = -(1/B) sum_j (log pi~_j + H_bar), H_bar = -m (auto temperature);
 8. Adam on each network with its own t, then Polyak theta'_i <- tau theta_i,new + (1-tau) theta'_i;
 9. statistics.

Readings used: #1 SAC v2 (twin target Qs, auto alpha),
#3 Jacobi order, #4 ReLU hidden / critic input [s | a], #5 constants,
#6 clamp gradient passes at the bounds inclusive, #7 stable squash correction,
#8 normalised action space, #9 tie-breaks, #10 loss scaling, #11 Adam form.
"""

from dataclasses import dataclass, field

import numpy as np

from . import mlp, optim, philox

LN2 = np.log(2.0)
HALF_LN_2PI = 0.5 * np.log(2.0 * np.pi)


@dataclass
class Config:
    obs_dim: int
    act_dim: int
    hidden: int = 256
    n_hidden: int = 2
    gamma: float = 0.99
    tau: float = 0.005
    lr_actor: float = 3e-4
    lr_critic: float = 3e-4
    lr_alpha: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    alpha_auto: bool = True
    alpha_init: float = 0.2
    target_entropy: float = None  # default -m
    log_std_min: float = -20.0
    log_std_max: float = 2.0
    # TD3 (reading #18)
    td3_noise: float = 0.2
    td3_noise_clip: float = 0.5
    td3_policy_delay: int = 2

    def __post_init__(self):
        if self.target_entropy is None:
            self.target_entropy = -float(self.act_dim)


def actor_shapes(cfg, td3=False):
    return mlp.layer_dims(cfg.obs_dim, cfg.hidden, cfg.n_hidden, cfg.act_dim if td3 else 2 * cfg.act_dim)


def critic_shapes(cfg):
    return mlp.layer_dims(cfg.obs_dim + cfg.act_dim, cfg.hidden, cfg.n_hidden, 1)


@dataclass
class State:
    """Flat float64 parameter vectors in the §8(b) layout plus optimizer state."""
    actor: np.ndarray
    q1: np.ndarray
    q2: np.ndarray
    q1_targ: np.ndarray
    q2_targ: np.ndarray
    log_alpha: float
    actor_targ: np.ndarray = None  # TD3 only
    opt: dict = field(default_factory=dict)
    step: int = 0

    @staticmethod
    def create(actor, q1, q2, q1_targ=None, q2_targ=None, log_alpha=0.0, actor_targ=None):
        f = lambda x: np.asarray(x, dtype=np.float64).copy()
        st = State(actor=f(actor), q1=f(q1), q2=f(q2),
                   q1_targ=f(q1 if q1_targ is None else q1_targ),
                   q2_targ=f(q2 if q2_targ is None else q2_targ),
                   log_alpha=float(log_alpha),
                   actor_targ=None if actor_targ is None else f(actor_targ))
        st.opt = {"actor": optim.AdamState(st.actor.size), "q1": optim.AdamState(st.q1.size),
                  "q2": optim.AdamState(st.q2.size), "alpha": optim.AdamState(1)}
        return st

    def copy(self):
        c = State(actor=self.actor.copy(), q1=self.q1.copy(), q2=self.q2.copy(),
                  q1_targ=self.q1_targ.copy(), q2_targ=self.q2_targ.copy(),
                  log_alpha=self.log_alpha,
                  actor_targ=None if self.actor_targ is None else self.actor_targ.copy(),
                  step=self.step)
        c.opt = {k: v.copy() for k, v in self.opt.items()}
        return c


# ----------------------------------------------------------------------------- policy head

def softplus(x):
    return np.maximum(x, 0.0) + np.log1p(np.exp(-np.abs(x)))


def sigmoid(x):
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def policy_forward(actor_params, s, eps, cfg, relu_masks=None):
    """Squashed-Gaussian policy (§8(c) step 3)."""
    m = cfg.act_dim
    H, cache = mlp.forward(actor_params, s, relu_masks)
    mu, l = H[:, :m], H[:, m:2 * m]
    lc = np.clip(l, cfg.log_std_min, cfg.log_std_max)
    sigma = np.exp(lc)
    u = mu + sigma * eps
    a = np.tanh(u)
    logp = np.sum(-0.5 * eps * eps - lc - HALF_LN_2PI - 2.0 * (LN2 - u - softplus(-2.0 * u)), axis=1)
    head = dict(l=l, lc=lc, sigma=sigma, u=u, a=a, eps=eps)
    return a, logp, cache, head


def policy_head_backward(head, g_a, g_lp, cfg):
    """Chain rule through the head, written step by step (reading #6, eq. H).

    g_a = dL/da [B x m], g_lp = dL/d log pi [B].  Returns dL/d[mu | l].
    """
    a, u, sigma, eps, l = head["a"], head["u"], head["sigma"], head["eps"], head["l"]
    g_lp = np.asarray(g_lp, dtype=np.float64).reshape(-1, 1)
    # a = tanh(u)
    g_u = g_a * (1.0 - a * a)
    # log pi contains -2 (ln 2 - u - softplus(-2u)); d/du = 2 - 4 sigmoid(-2u)
    g_u = g_u + g_lp * (2.0 - 4.0 * sigmoid(-2.0 * u))
    # u = mu + sigma * eps
    g_mu = g_u
    g_sigma = g_u * eps
    # sigma = exp(lc); log pi contains -lc
    g_lc = g_sigma * sigma - g_lp
    # lc = clamp(l, lo, hi): gradient passes where lo <= l <= hi (inclusive)
    g_l = g_lc * ((l >= cfg.log_std_min) & (l <= cfg.log_std_max))
    return np.concatenate([g_mu, g_l], axis=1)


def critic_q(params, s, a, relu_masks=None):
    q, cache = mlp.forward(params, np.concatenate([s, a], axis=1), relu_masks)
    return q[:, 0], cache


# ----------------------------------------------------------------------------- gradients

def _batch_f64(batch):
    return (np.asarray(batch["obs"], np.float64), np.asarray(batch["act"], np.float64),
            np.asarray(batch["rew"], np.float64), np.asarray(batch["next_obs"], np.float64),
            np.asarray(batch["done"], np.float64))


def min_weights(q1, q2):
    """(w1, w2) = (1,0) if q1<q2, (0,1) if q2<q1, (1/2,1/2) on a tie (reading #9)."""
    w1 = np.where(q1 < q2, 1.0, np.where(q1 > q2, 0.0, 0.5))
    return w1, 1.0 - w1


def sac_grads(st, batch, eps, eps2, cfg, B_global, critic=True, actor=True, decisions=None):
    """Gradients of L_Q (critics), L_pi (actor) and L_alpha over the given rows.

    Every row contributes with the global 1/B, so gradients of row shards add
    up exactly.  Returns (grads, sums) where sums holds the
    row sums behind the reported statistics.

    decisions (optional; reading #25): the comparisons a floating-point value decides,
    taken by the kernel in its precision and used here instead of this oracle's own -- ReLU masks
    "q1"/"q2" (online critics on the loss rows), "q1_pi"/"q2_pi" (on the actor rows), "actor" (the
    actor on s), and "w1" (the min-tie weight of Q1 on the actor rows).  Absent keys: own decisions.
    """
    dec = decisions or {}
    s, a, r, s2, d = _batch_f64(batch)
    m, o = cfg.act_dim, cfg.obs_dim
    alpha = np.exp(st.log_alpha)
    A = mlp.unflatten(st.actor, actor_shapes(cfg))
    cs = critic_shapes(cfg)
    Q = [mlp.unflatten(st.q1, cs), mlp.unflatten(st.q2, cs)]
    grads, sums = {}, {}
    if critic:
        a2, logp2, _, _ = policy_forward(A, s2, eps2, cfg)
        qt1, _ = critic_q(mlp.unflatten(st.q1_targ, cs), s2, a2)
        qt2, _ = critic_q(mlp.unflatten(st.q2_targ, cs), s2, a2)
        y = r + cfg.gamma * (1.0 - d) * (np.minimum(qt1, qt2) - alpha * logp2)
        lq = 0.0
        for i in range(2):
            q, cache = critic_q(Q[i], s, a, dec.get(f"q{i + 1}"))
            dq = 2.0 * (q - y) / B_global
            g, _ = mlp.backward(Q[i], cache, dq.reshape(-1, 1))
            grads[f"q{i + 1}"] = mlp.flatten(g)
            lq = lq + np.sum((q - y) ** 2)
            sums[f"q{i + 1}"] = np.sum(q)
            sums[f"q{i + 1}_abs"] = np.sum(np.abs(q))  # conditioning of the mean (test tolerance scale)
        sums["lq"] = lq
        sums["y"] = y
    if actor:
        at, logpt, acache, head = policy_forward(A, s, eps, cfg, dec.get("actor"))
        qs, caches = [], []
        for i in range(2):
            q, cache = critic_q(Q[i], s, at, dec.get(f"q{i + 1}_pi"))
            qs.append(q)
            caches.append(cache)
        w1, w2 = min_weights(qs[0], qs[1])
        if "w1" in dec:
            w1 = np.asarray(dec["w1"], np.float64)
            w2 = 1.0 - w1
        g_a = np.zeros_like(at)
        for i, w in enumerate((w1, w2)):
            dq = -w / B_global
            _, dX = mlp.backward(Q[i], caches[i], dq.reshape(-1, 1))
            g_a += dX[:, o:o + m]
        g_lp = np.full(s.shape[0], alpha / B_global)
        dH = policy_head_backward(head, g_a, g_lp, cfg)
        g, _ = mlp.backward(A, acache, dH)
        grads["actor"] = mlp.flatten(g)
        if cfg.alpha_auto:
            grads["log_alpha"] = np.array([-np.sum(logpt + cfg.target_entropy) / B_global])
        sums["lpi"] = np.sum(alpha * logpt - np.minimum(qs[0], qs[1]))
        sums["lpi_abs"] = np.sum(np.abs(alpha * logpt - np.minimum(qs[0], qs[1])))  # conditioning of the mean
        sums["logp"] = np.sum(logpt)
    return grads, sums


def sac_apply(st, grads, cfg, critic=True, actor=True):
    """Adam on every trained network (own t each), then Polyak on the targets."""
    st = st.copy()
    adam = lambda th, g, key, lr: optim.adam_step(th, g, st.opt[key], lr, cfg.beta1, cfg.beta2, cfg.adam_eps)
    if critic:
        st.q1 = adam(st.q1, grads["q1"], "q1", cfg.lr_critic)
        st.q2 = adam(st.q2, grads["q2"], "q2", cfg.lr_critic)
        st.q1_targ = optim.polyak(st.q1_targ, st.q1, cfg.tau)
        st.q2_targ = optim.polyak(st.q2_targ, st.q2, cfg.tau)
    if actor:
        st.actor = adam(st.actor, grads["actor"], "actor", cfg.lr_actor)
        if cfg.alpha_auto:
            st.log_alpha = float(adam(np.array([st.log_alpha]), grads["log_alpha"], "alpha", cfg.lr_alpha)[0])
    st.step += 1
    return st


def stats_of(st, sums, B, cfg):
    alpha = float(np.exp(st.log_alpha))
    return dict(
        step=st.step,
        critic_loss=float(sums["lq"] / B),
        actor_loss=float(sums["lpi"] / B),
        actor_loss_abs=float(sums.get("lpi_abs", 0.0) / B),
        alpha=alpha,
        alpha_loss=float(-st.log_alpha * (sums["logp"] / B + cfg.target_entropy)),
        q1_mean=float(sums["q1"] / B),
        q2_mean=float(sums["q2"] / B),
        q1_mean_abs=float(sums.get("q1_abs", 0.0) / B),
        q2_mean_abs=float(sums.get("q2_abs", 0.0) / B),
        logp_mean=float(sums["logp"] / B),
    )


def draw_noise(seed, step, batch, m, row0=0):
    eps = philox.normals(seed, step, philox.S_EPS, batch, m, row0=row0)
    eps2 = philox.normals(seed, step, philox.S_EPS2, batch, m, row0=row0)
    return eps, eps2


def sac_step(st, ring, B, seed, cfg):
    """One full single-device SAC update at step k = st.step.  Returns (state', stats, idx)."""
    k = st.step
    idx, batch = ring.sample(B, seed, k)
    eps, eps2 = draw_noise(seed, k, B, cfg.act_dim)
    grads, sums = sac_grads(st, batch, eps, eps2, cfg, B)
    stats = stats_of(st, sums, B, cfg)
    return sac_apply(st, grads, cfg), stats, idx
