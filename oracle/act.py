"""Sampler-side action selection from a synced actor, float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3.2.1: the sampling processes' actions are "generate[d] ... by forward propagation"
of the policy; §3.2.2: the test process acts deterministically.  The policy is the actor
of oracle/sac.py (squashed Gaussian) or oracle/td3.py (tanh):

  SAC, deterministic:  a = tanh(mu)
  SAC, stochastic:     a = tanh(mu + exp(clamp(l, lo, hi)) * n)            (the reparameterised sample)
  TD3, deterministic:  a = tanh(z)
  TD3, stochastic:     a = clip(tanh(z) + sigma_x * n, -1, 1)              (Gaussian exploration)

with [mu | l] (SAC) or z (TD3) = MLP_phi(s) and n[j, i] = philox.normals(seed, step, S_ACT, ...)
for row j of the call.  Readings: S_ACT = 7 (a new Philox stream id; 6 is reserved for
synthetic data in SURVEY.md §8(c) #13); sigma_x = 0.1 (Fujimoto et al.'s exploration noise; the
paper is silent); actions stay in the normalised [-1, 1] space (reading #8).
"""

import numpy as np

from . import mlp, philox
from .sac import actor_shapes

S_ACT = 7


def act(actor_flat, obs, cfg, algo="sac", deterministic=False, seed=0, step=0, expl_noise=0.1):
    """Actions [n x m] of the flat actor `actor_flat` (§8(b) layout) on observations obs [n x o]."""
    td3 = algo == "td3"
    m = cfg.act_dim
    A = mlp.unflatten(actor_flat, actor_shapes(cfg, td3=td3))
    H, _ = mlp.forward(A, np.asarray(obs, dtype=np.float64))
    n = H.shape[0]
    if not td3:
        mu, l = H[:, :m], H[:, m:2 * m]
        if deterministic:
            return np.tanh(mu)
        eps = philox.normals(seed, step, S_ACT, n, m)
        return np.tanh(mu + np.exp(np.clip(l, cfg.log_std_min, cfg.log_std_max)) * eps)
    a = np.tanh(H)
    if deterministic:
        return a
    noise = philox.normals(seed, step, S_ACT, n, m)
    return np.clip(a + expl_noise * noise, -1.0, 1.0)
