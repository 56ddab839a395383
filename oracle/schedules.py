"""The two parallel schedules of the update, as reorganisations of the single one.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``sharded_step``: the G-way row-sharded (data-parallel) schedule
  (Fig. 2(a) ``fig_multi_gpu``(a)): global rows
  [0, B) split contiguously; each shard draws its own rows' indices and noise
  from the same counters, computes gradients scaled by the global 1/B, and the
  shard gradients are summed (the allreduce) before one identical Adam step.
* ``split_step``: the actor/critic split (Fig. 3 ``fig_update``):
  the critic side computes the critic update from a copy of phi_k and alpha_k,
  the actor side computes the actor + temperature update from copies of
  theta_1,k and theta_2,k (Jacobi, reading #3); parameters are then exchanged.

tests/test_oracle_schedules.py asserts both equal ``sac.sac_step`` /
``td3.td3_step`` to 1e-12 relative in float64.
"""

import numpy as np

from . import sac, td3


def _shards(B, G):
    base, rem = divmod(B, G)
    out, r0 = [], 0
    for g in range(G):
        n = base + (1 if g < rem else 0)
        out.append((r0, n))
        r0 += n
    return out


def _sum_dicts(ds):
    out = {}
    for d in ds:
        for k, v in d.items():
            if k == "y":
                out[k] = np.concatenate([out[k], v]) if k in out else v
            else:
                out[k] = out[k] + v if k in out else v
    return out


def sharded_step(st, ring, B, seed, cfg, G, algo="sac"):
    k = st.step
    gs, ss, idxs = [], [], []
    for r0, n in _shards(B, G):
        idx, batch = ring.sample(n, seed, k, row0=r0, global_batch=B)
        idxs.append(idx)
        if algo == "sac":
            eps, eps2 = sac.draw_noise(seed, k, n, cfg.act_dim, row0=r0)
            g, s = sac.sac_grads(st, batch, eps, eps2, cfg, B)
        else:
            xi = td3.draw_smoothing(seed, k, n, cfg, row0=r0)
            g, s = td3.td3_grads(st, batch, xi, cfg, B, k)
        gs.append(g)
        ss.append(s)
    grads, sums = _sum_dicts(gs), _sum_dicts(ss)
    if algo == "sac":
        stats = sac.stats_of(st, sums, B, cfg)
        return sac.sac_apply(st, grads, cfg), stats, np.concatenate(idxs)
    stats = td3.stats_of(st, sums, B)
    return td3.td3_apply(st, grads, cfg, k), stats, np.concatenate(idxs)


def split_step(st, ring, B, seed, cfg, algo="sac"):
    """Critic side and actor side each work on private copies of step-k state."""
    k = st.step
    critic_side, actor_side = st.copy(), st.copy()
    idx, batch = ring.sample(B, seed, k)
    if algo == "sac":
        eps, eps2 = sac.draw_noise(seed, k, B, cfg.act_dim)
        gc, sc = sac.sac_grads(critic_side, batch, None, eps2, cfg, B, critic=True, actor=False)
        ga, sa = sac.sac_grads(actor_side, batch, eps, None, cfg, B, critic=False, actor=True)
        critic_side = sac.sac_apply(critic_side, gc, cfg, critic=True, actor=False)
        actor_side = sac.sac_apply(actor_side, ga, cfg, critic=False, actor=True)
        stats = sac.stats_of(st, {**sc, **sa}, B, cfg)
    else:
        xi = td3.draw_smoothing(seed, k, B, cfg)
        gc, sc = td3.td3_grads(critic_side, batch, xi, cfg, B, k, critic=True, actor=False)
        ga, sa = td3.td3_grads(actor_side, batch, None, cfg, B, k, critic=False, actor=True)
        critic_side = td3.td3_apply(critic_side, gc, cfg, k, critic=True, actor=False)
        actor_side = td3.td3_apply(actor_side, ga, cfg, k, critic=False, actor=True)
        stats = td3.stats_of(st, {**sc, **sa}, B)
    # parameter exchange at the step boundary (a10): each side takes the other's networks
    out = critic_side
    out.actor = actor_side.actor
    out.log_alpha = actor_side.log_alpha
    out.opt["actor"] = actor_side.opt["actor"]
    out.opt["alpha"] = actor_side.opt["alpha"]
    if algo == "td3":
        out.actor_targ = actor_side.actor_targ
    return out, stats, idx
