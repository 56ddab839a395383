"""Pins for oracle/mlp.py: S:52-54 (forward), S:61-63 and S:84 (backward)."""

import numpy as np
import pytest
import torch

from oracle import mlp


def _rand_net(rng, dims):
    return [(rng.standard_normal((o, i)), rng.standard_normal(o)) for o, i in zip(dims[1:], dims[:-1])]


def test_zero_net_gives_zero():
    P = [(np.zeros((5, 4)), np.zeros(5)), (np.zeros((2, 5)), np.zeros(2))]
    y, _ = mlp.forward(P, np.random.default_rng(0).standard_normal((7, 4)))
    assert np.array_equal(y, np.zeros((7, 2)))


def test_identity_layer():
    X = np.random.default_rng(1).standard_normal((6, 4))
    y, _ = mlp.forward([(np.eye(4), np.zeros(4))], X)
    assert np.array_equal(y, X)


def test_hand_computed_two_layer_3x4():
    # seeded 2-layer net on a 3x4 input vs an independent hand computation.
    X = np.array([[1, 2, 0, -1], [0, 1, 1, 1], [2, -1, 0, 3]], dtype=np.float64)
    W1 = np.array([[1, 0, -1, 1], [0, 2, 1, -1]], dtype=np.float64)
    b1 = np.array([0.5, -1.0])
    W2 = np.array([[2, -3]], dtype=np.float64)
    b2 = np.array([1.0])
    # row 1: z1 = (0.5, 4)   -> 2*0.5 - 3*4 + 1 = -10
    # row 2: z1 = (0.5, 1)   -> 1 - 3 + 1       = -1
    # row 3: z1 = (5.5, -6)  -> relu (5.5, 0)   -> 11 + 1 = 12
    y, _ = mlp.forward([(W1, b1), (W2, b2)], X)
    assert np.array_equal(y[:, 0], [-10.0, -1.0, 12.0])


def test_linear_case_closed_form():
    # loss = sum(outputs), linear net -> dW = X^T 1 (per output row), db = B
    rng = np.random.default_rng(2)
    X = rng.standard_normal((9, 4))
    P = [(rng.standard_normal((3, 4)), rng.standard_normal(3))]
    y, cache = mlp.forward(P, X)
    g, dX = mlp.backward(P, cache, np.ones_like(y))
    assert np.allclose(g[0][0], np.tile(X.sum(0), (3, 1)), rtol=0, atol=1e-12)
    assert np.array_equal(g[0][1], np.full(3, 9.0))
    assert np.allclose(dX, np.tile(P[0][0].sum(0), (9, 1)), atol=1e-12)


def test_zero_adjoint_gives_zero_gradients():
    rng = np.random.default_rng(3)
    P = _rand_net(rng, [4, 8, 8, 2])
    y, cache = mlp.forward(P, rng.standard_normal((5, 4)))
    g, dX = mlp.backward(P, cache, np.zeros_like(y))
    assert all(not np.any(dW) and not np.any(db) for dW, db in g) and not np.any(dX)


@pytest.mark.parametrize("dims", [[3, 5, 2], [4, 16, 16, 1], [6, 7, 9, 3], [2, 16, 16, 16, 4]])
def test_central_finite_differences(dims):
    # step 1e-5, relative 1e-6 in fp64 (1e-6 absolute floor), every parameter
    rng = np.random.default_rng(sum(dims))
    P = _rand_net(rng, dims)
    X = rng.standard_normal((7, dims[0]))
    C = rng.standard_normal((7, dims[-1]))  # L = sum(C * Y)
    y, cache = mlp.forward(P, X)
    g, dX = mlp.backward(P, cache, C)
    flat = mlp.flatten(P)
    shapes = [(o, i) for o, i in zip(dims[1:], dims[:-1])]
    gflat = mlp.flatten(g)
    h = 1e-5
    for p in range(flat.size):
        e = np.zeros_like(flat)
        e[p] = h
        lp = np.sum(C * mlp.forward(mlp.unflatten(flat + e, shapes), X)[0])
        lm = np.sum(C * mlp.forward(mlp.unflatten(flat - e, shapes), X)[0])
        fd = (lp - lm) / (2 * h)
        assert abs(fd - gflat[p]) <= 1e-6 * max(abs(fd), 1.0), (p, fd, gflat[p])


def test_torch_autograd_float64_cross_check():
    rng = np.random.default_rng(11)
    dims = [10, 32, 32, 5]
    P = _rand_net(rng, dims)
    X = rng.standard_normal((13, 10))
    C = rng.standard_normal((13, 5))
    y, cache = mlp.forward(P, X)
    g, dX = mlp.backward(P, cache, C)
    tp = [(torch.tensor(W, requires_grad=True), torch.tensor(b, requires_grad=True)) for W, b in P]
    tx = torch.tensor(X, requires_grad=True)
    a = tx
    for l, (W, b) in enumerate(tp):
        a = torch.nn.functional.linear(a, W, b)
        if l < len(tp) - 1:
            a = torch.relu(a)
    (a * torch.tensor(C)).sum().backward()
    assert np.allclose(y, a.detach().numpy(), rtol=1e-13, atol=1e-13)
    for (dW, db), (W, b) in zip(g, tp):
        assert np.allclose(dW, W.grad.numpy(), rtol=1e-12, atol=1e-12)
        assert np.allclose(db, b.grad.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(dX, tx.grad.numpy(), rtol=1e-12, atol=1e-12)


def test_flat_roundtrip_and_layout():
    rng = np.random.default_rng(5)
    shapes = mlp.layer_dims(3, 4, 2, 2)
    assert shapes == [(4, 3), (4, 4), (2, 4)]
    flat = rng.standard_normal(mlp.n_params(shapes))
    P = mlp.unflatten(flat, shapes)
    assert np.array_equal(mlp.flatten(P), flat)
    # W1 is row-major [out x in] at offset 0, b1 follows
    assert np.array_equal(P[0][0].ravel(), flat[:12]) and np.array_equal(P[0][1], flat[12:16])
