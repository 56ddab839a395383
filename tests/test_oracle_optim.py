"""Pins for oracle/optim.py: Adam and Polyak."""

import numpy as np
import torch

from oracle import optim


def test_adam_zero_gradient_noop_and_counter():
    th = np.array([1.0, -2.0, 3.0])
    st = optim.AdamState(3)
    out = optim.adam_step(th, np.zeros(3), st, lr=1e-3)
    assert np.array_equal(out, th) and st.t == 1


def test_adam_first_step_closed_form():
    # bias-corrected moments cancel: delta = -lr * g / (|g| + eps)
    g = np.array([1e-9, -3.0, 0.25, 7e3])
    st = optim.AdamState(4)
    out = optim.adam_step(np.zeros(4), g, st, lr=1e-3, eps=1e-8)
    assert np.allclose(out, -1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-14, atol=0)


def test_adam_constant_gradient_constant_step():
    # m_hat = g and v_hat = g^2 for a constant g, so every step is identical
    g = np.array([0.3, -1.5])
    st = optim.AdamState(2)
    th = np.zeros(2)
    prev = th
    for t in range(25):
        th = optim.adam_step(th, g, st, lr=1e-2)
        assert np.allclose(th - prev, -1e-2 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=1e-15)
        prev = th


def test_adam_quadratic_convergence():
    # 1000 steps on f(x) = x^2 from x = 1 with lr 1e-2 -> |x| < 0.05
    st = optim.AdamState(1)
    x = np.array([1.0])
    for _ in range(1000):
        x = optim.adam_step(x, 2 * x, st, lr=1e-2)
    assert abs(x[0]) < 0.05


def test_adam_matches_torch_adam_float64():
    rng = np.random.default_rng(0)
    th0 = rng.standard_normal(50)
    p = torch.tensor(th0.copy(), requires_grad=True)
    opt = torch.optim.Adam([p], lr=3e-4, betas=(0.9, 0.999), eps=1e-8)
    st = optim.AdamState(50)
    th = th0.copy()
    for k in range(7):
        g = rng.standard_normal(50) * 10.0 ** rng.integers(-6, 2, 50)
        p.grad = torch.tensor(g)
        opt.step()
        th = optim.adam_step(th, g, st, lr=3e-4)
    assert np.allclose(th, p.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_polyak_bounds_and_geometric_decay():
    rng = np.random.default_rng(1)
    t0, th = rng.standard_normal(10), rng.standard_normal(10)
    assert np.array_equal(optim.polyak(t0, th, 0.0), t0)
    assert np.array_equal(optim.polyak(t0, th, 1.0), th)
    tau, t = 0.005, t0
    for n in range(1, 201):
        t = optim.polyak(t, th, tau)
    assert np.allclose(t - th, (1 - tau) ** 200 * (t0 - th), rtol=1e-12, atol=1e-15)
