"""Seeded synthetic inputs shared (as data) by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws replay
transitions shaped like the paper's tasks and initial network parameters,
from numpy's PCG64.  Both ``oracle/`` (via tests and bench) and the product
path receive the same arrays; neither side's code lives here.

Workloads (BASELINE.json ``configs``; SURVEY.md §8(d) "Synthetic inputs"):

* PEN  -- Pendulum-shaped SAC: obs 3, act 1, 2x64, B 256, ring 10K.  Physically
          consistent rows: theta ~ U(-pi, pi), theta_dot ~ U(-8, 8),
          s = (cos, sin, theta_dot), a ~ U(-1, 1) (torque 2a), one step of the
          Pendulum dynamics (g 10, m = l = 1, dt 0.05, speed clip 8),
          r = -(theta^2 + 0.1 theta_dot^2 + 0.001 torque^2), d = 0.
* WLK  -- Walker2d-shaped SAC: obs 22, act 6, 2x256, B 8192, ring 1M.
* ANT  -- Ant-shaped SAC: obs 28, act 8, 2x256, B 32768, ring 1M.
* HUM  -- Humanoid-shaped SAC: obs 44, act 17, 3x512, B 65536, ring 1M.
* TD3  -- Humanoid-shaped TD3: obs 44, act 17, 3x1024, B 131072, ring 4M.

Locomotion rows: s ~ clip(N(0,1), +-5), s2 = clip(s + 0.1 N(0,1), +-5),
a ~ U(-0.999, 0.999), r ~ N(0,1), d ~ Bernoulli(0.01).

Seeds: data 2312, sample 6126, init 0.
"""

from dataclasses import dataclass

import numpy as np

DATA_SEED = 2312
SAMPLE_SEED = 6126
INIT_SEED = 0


@dataclass(frozen=True)
class Workload:
    name: str
    algo: str  # "sac" | "td3"
    obs_dim: int
    act_dim: int
    hidden: int
    n_hidden: int
    batch: int
    capacity: int
    kind: str  # "pendulum" | "locomotion"


WORKLOADS = {
    "pendulum": Workload("pendulum", "sac", 3, 1, 64, 2, 256, 10_000, "pendulum"),
    "walker": Workload("walker", "sac", 22, 6, 256, 2, 8192, 1_000_000, "locomotion"),
    "ant": Workload("ant", "sac", 28, 8, 256, 2, 32768, 1_000_000, "locomotion"),
    "humanoid": Workload("humanoid", "sac", 44, 17, 512, 3, 65536, 1_000_000, "locomotion"),
    "humanoid_td3": Workload("humanoid_td3", "td3", 44, 17, 1024, 3, 131072, 4_000_000, "locomotion"),
}


def transitions(kind, obs_dim, act_dim, n, seed=DATA_SEED):
    """n synthetic transitions -> dict of float32 arrays obs, act, rew, next_obs, done."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "pendulum":
        assert obs_dim == 3 and act_dim == 1
        th = rng.uniform(-np.pi, np.pi, n)
        thd = rng.uniform(-8.0, 8.0, n)
        a = rng.uniform(-1.0, 1.0, n)
        torque = 2.0 * a
        g, mass, length, dt = 10.0, 1.0, 1.0, 0.05
        r = -(th ** 2 + 0.1 * thd ** 2 + 0.001 * torque ** 2)
        thd2 = thd + (3.0 * g / (2.0 * length) * np.sin(th) + 3.0 / (mass * length ** 2) * torque) * dt
        thd2 = np.clip(thd2, -8.0, 8.0)
        th2 = th + thd2 * dt
        obs = np.stack([np.cos(th), np.sin(th), thd], 1)
        nobs = np.stack([np.cos(th2), np.sin(th2), thd2], 1)
        return dict(obs=obs.astype(np.float32), act=a.reshape(-1, 1).astype(np.float32),
                    rew=r.astype(np.float32), next_obs=nobs.astype(np.float32),
                    done=np.zeros(n, np.float32))
    s = np.clip(rng.standard_normal((n, obs_dim)), -5, 5)
    s2 = np.clip(s + 0.1 * rng.standard_normal((n, obs_dim)), -5, 5)
    a = rng.uniform(-0.999, 0.999, (n, act_dim))
    r = rng.standard_normal(n)
    d = (rng.random(n) < 0.01).astype(np.float64)
    return dict(obs=s.astype(np.float32), act=a.astype(np.float32), rew=r.astype(np.float32),
                next_obs=s2.astype(np.float32), done=d.astype(np.float32))


def workload_transitions(w: Workload, n=None, seed=DATA_SEED):
    return transitions(w.kind, w.obs_dim, w.act_dim, w.capacity if n is None else n, seed)


def layer_shapes(in_dim, hidden, n_hidden, out_dim):
    dims = [in_dim] + [hidden] * n_hidden + [out_dim]
    return list(zip(dims[1:], dims[:-1]))


def init_flat(shapes, seed=INIT_SEED, stream=0):
    """nn.Linear-default init W, b ~ U(+-1/sqrt(fan_in)) as a flat float32 vector [W1|b1|W2|b2...]."""
    rng = np.random.Generator(np.random.PCG64([seed, stream]))
    parts = []
    for o, i in shapes:
        bound = 1.0 / np.sqrt(i)
        parts.append(rng.uniform(-bound, bound, o * i))
        parts.append(rng.uniform(-bound, bound, o))
    return np.concatenate(parts).astype(np.float32)


def init_params(obs_dim, act_dim, hidden, n_hidden, algo="sac", seed=INIT_SEED):
    """Initial actor / critic parameter vectors (targets copy the online nets)."""
    a_out = 2 * act_dim if algo in ("sac", "sacv1") else act_dim
    actor = init_flat(layer_shapes(obs_dim, hidden, n_hidden, a_out), seed, 1)
    cs = layer_shapes(obs_dim + act_dim, hidden, n_hidden, 1)
    q1 = init_flat(cs, seed, 2)
    q2 = init_flat(cs, seed, 3)
    out = dict(actor=actor, q1=q1, q2=q2)
    if algo == "sacv1":  # + the state-value network V(s)
        out["v"] = init_flat(layer_shapes(obs_dim, hidden, n_hidden, 1), seed, 4)
    return out
