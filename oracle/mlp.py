"""Dense ReLU MLP: forward and manual reverse-mode backward, float64 (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SPEC nn-core forward/backward: a stack of affine layers, hidden
layers followed by ReLU (reading #4: north_star "bias, ReLU"; the paper is
silent on the activation), linear output.  Parameters per layer are
W [out x in] (the nn.Linear convention) and b [out]; the flat layout is
W_1, b_1, W_2, b_2, ... (SURVEY.md §8(b) "Flat layout").

ReLU'(0) = 0 (reading #9).  Pinned by tests/test_oracle_mlp.py: zero net,
identity layer, a hand-computed 2-layer example, the linear-case
closed form dW = X^T 1, central finite differences and a
torch.autograd float64 cross-check.
"""

import numpy as np


def layer_dims(in_dim, hidden, n_hidden, out_dim):
    dims = [in_dim] + [hidden] * n_hidden + [out_dim]
    return list(zip(dims[1:], dims[:-1]))  # (out, in) per layer


def n_params(shapes):
    return sum(o * i + o for o, i in shapes)


def unflatten(flat, shapes):
    """Flat [W1 | b1 | W2 | b2 | ...] -> list of (W, b) float64 views/copies."""
    flat = np.asarray(flat, dtype=np.float64)
    out, p = [], 0
    for o, i in shapes:
        W = flat[p:p + o * i].reshape(o, i)
        p += o * i
        b = flat[p:p + o]
        p += o
        out.append((W.copy(), b.copy()))
    assert p == flat.size, (p, flat.size)
    return out


def flatten(params):
    return np.concatenate([np.concatenate([W.ravel(), b.ravel()]) for W, b in params])


def forward(params, X, relu_masks=None):
    """Returns (output, cache).  cache = list of layer inputs, pre-activations and ReLU decisions.

    relu_masks (optional, one boolean [rows x out] array per hidden layer): the ReLU decisions
    1[Z > 0] taken elsewhere -- by the kernel, in its precision -- and used here in place of this
    function's own fp64 comparison (the task's rule for decisions a floating-point value takes;
    DESIGN.md reading #25).  None: the plain ReLU."""
    A = np.asarray(X, dtype=np.float64)
    cache = []
    L = len(params)
    for l, (W, b) in enumerate(params):
        Z = A @ W.T + b
        if l < L - 1:
            mask = (Z > 0.0) if relu_masks is None else np.asarray(relu_masks[l], dtype=bool)
            cache.append((A, Z, mask))
            A = np.where(mask, Z, 0.0)
        else:
            cache.append((A, Z, None))
            A = Z
    return A, cache


def backward(params, cache, dY):
    """Reverse-mode: given dL/dY returns (grads [(dW, db)], dL/dX)."""
    L = len(params)
    grads = [None] * L
    dZ = np.asarray(dY, dtype=np.float64)
    for l in range(L - 1, -1, -1):
        W, _ = params[l]
        A_in = cache[l][0]
        grads[l] = (dZ.T @ A_in, dZ.sum(axis=0))
        dA = dZ @ W
        if l > 0:
            dZ = dA * cache[l - 1][2]  # ReLU'(Z) = 1[Z > 0] (ReLU'(0) = 0)
        else:
            dX = dA
    return grads, dX
