"""Pins for oracle/act.py (sampler-side action selection)."""

import numpy as np
import pytest

import synthdata
from oracle import act, mlp, philox, sac


def _head_only_actor(o, m, h, L, b_head, td3=False):
    """Every weight zero, hidden biases zero: the MLP output is the head bias for every row."""
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L)
    shapes = sac.actor_shapes(cfg, td3=td3)
    flat = np.zeros(mlp.n_params(shapes))
    flat[-shapes[-1][0]:] = b_head
    return cfg, flat


def test_sac_closed_form_on_a_bias_only_actor():
    o, m, n = 4, 3, 9
    mu, l = np.array([0.3, -1.2, 2.0]), np.array([-0.5, 0.4, -30.0])  # last log sigma below the clamp
    cfg, flat = _head_only_actor(o, m, 8, 2, np.concatenate([mu, l]))
    s = np.random.default_rng(0).normal(size=(n, o))
    det = act.act(flat, s, cfg, deterministic=True)
    assert np.array_equal(det, np.tile(np.tanh(mu), (n, 1)))
    sto = act.act(flat, s, cfg, deterministic=False, seed=11, step=5)
    eps = philox.normals(11, 5, act.S_ACT, n, m)
    sig = np.exp(np.array([-0.5, 0.4, -20.0]))  # clamp to [-20, 2]
    assert np.allclose(sto, np.tanh(mu + sig * eps), rtol=0, atol=1e-15)


def test_sac_tiny_sigma_is_deterministic_and_matches_policy_forward():
    o, m, h, L, n = 5, 2, 16, 2, 50
    cfg = sac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L)
    flat = synthdata.init_params(o, m, h, L, seed=3)["actor"].astype(np.float64)
    s = np.random.default_rng(1).normal(size=(n, o))
    # the stochastic action is exactly the training path's reparameterised sample with eps from S_ACT
    eps = philox.normals(7, 2, act.S_ACT, n, m)
    a_train, _, _, _ = sac.policy_forward(mlp.unflatten(flat, sac.actor_shapes(cfg)), s, eps, cfg)
    assert np.allclose(act.act(flat, s, cfg, seed=7, step=2), a_train, rtol=0, atol=1e-15)
    # log sigma pushed to the lower clamp: sigma = e^-20, the sample collapses onto tanh(mu)
    shapes = sac.actor_shapes(cfg)
    Wl = flat.copy()
    nW = shapes[-1][0] * shapes[-1][1]
    head_w = Wl[-(nW + shapes[-1][0]):-shapes[-1][0]].reshape(shapes[-1])
    head_w[m:, :] = 0.0
    Wl[-(nW + shapes[-1][0]):-shapes[-1][0]] = head_w.ravel()
    Wl[-m:] = -50.0
    assert np.allclose(act.act(Wl, s, cfg, seed=7, step=2), act.act(Wl, s, cfg, deterministic=True), atol=1e-7)


def test_td3_clip_and_noise_scale():
    o, m, n = 3, 4, 20000
    cfg, flat = _head_only_actor(o, m, 8, 1, np.array([0.0, 0.5, -3.0, 30.0]), td3=True)
    s = np.zeros((n, o))
    det = act.act(flat, s, cfg, algo="td3", deterministic=True)
    assert np.allclose(det[0], np.tanh([0.0, 0.5, -3.0, 30.0]))
    sto = act.act(flat, s, cfg, algo="td3", seed=4, step=9, expl_noise=0.1)
    assert sto.min() >= -1.0 and sto.max() <= 1.0
    # column 0: tanh(0) + 0.1 n is never clipped here (|0.1 n| < 1): std 0.1 within 4 sigma of its estimate
    assert abs(sto[:, 0].std() - 0.1) < 4 * 0.1 / np.sqrt(2 * n)
    assert abs(sto[:, 0].mean()) < 4 * 0.1 / np.sqrt(n)
    # column 3: tanh(30) = 1 in float64, so every positive draw clips to exactly 1
    noise = philox.normals(4, 9, act.S_ACT, n, m)
    assert np.array_equal(sto[:, 3] == 1.0, noise[:, 3] >= 0)


def test_streams_and_rows_are_independent_draws():
    o, m, n = 3, 2, 4000
    cfg, flat = _head_only_actor(o, m, 8, 1, np.array([0.0, 0.0, 0.0, 0.0]))
    a1 = act.act(flat, np.zeros((n, o)), cfg, seed=1, step=0)
    a2 = act.act(flat, np.zeros((n, o)), cfg, seed=1, step=1)
    u1, u2 = np.arctanh(a1), np.arctanh(a2)
    # sigma = 1: u = eps ~ N(0, 1); consecutive steps uncorrelated
    assert abs(np.corrcoef(u1[:, 0], u2[:, 0])[0, 1]) < 4 / np.sqrt(n)
    assert abs(u1.std() - 1.0) < 0.05
