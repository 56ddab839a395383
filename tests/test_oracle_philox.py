"""Pins for oracle/philox.py (random numbers the update draws)."""

import os

import numpy as np
import pytest

from oracle import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    rows = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expected", _kat())
def test_philox_known_answer_vectors(ctr, key, expected):
    out = philox.philox4x32_10(*ctr, *key)
    assert [int(x) for x in out] == expected


def test_philox_vectorised_equals_scalar():
    j = np.arange(17, dtype=np.uint64)
    xs = philox.philox4x32_10(j, 3, 9, philox.S_EPS, 123, 456)
    for t in range(17):
        one = philox.philox4x32_10(t, 3, 9, philox.S_EPS, 123, 456)
        assert [int(x[t]) for x in xs] == [int(y) for y in one]


def _idx_alt(seed, step, F, B):
    """Independent evaluation of floor(X F / 2^64) via 32-bit limbs:
    X F = 2^32 (x1 F) + x0 F, so the quotient is floor((x1 F + floor(x0 F / 2^32)) / 2^32)."""
    k0, k1 = philox.key_of(seed)
    x0, x1, _, _ = philox.philox4x32_10(np.arange(B, dtype=np.uint64), 0, step, philox.S_IDX, k0, k1)
    p0 = x0.astype(np.uint64) * np.uint64(F)
    p1 = x1.astype(np.uint64) * np.uint64(F)
    return ((p1 + (p0 >> np.uint64(32))) >> np.uint64(32)).astype(np.int64)


@pytest.mark.parametrize("F", [1, 2, 3, 100, 10_000, 999_983, 1_000_000, 4_000_000, 2**31 - 1])
def test_index_map_limb_decomposition(F):
    idx = philox.sample_indices(6126, 5, F, 4096)
    assert np.array_equal(idx, _idx_alt(6126, 5, F, 4096))
    assert idx.min() >= 0 and idx.max() < F


def test_index_map_closed_forms():
    # F = 1 -> always slot 0 ("fill 1, B 1 -> that single record")
    assert np.all(philox.sample_indices(1, 0, 1, 1000) == 0)
    # F = 2^n -> the top n bits of X = x1 2^32 + x0
    k0, k1 = philox.key_of(77)
    x0, x1, _, _ = philox.philox4x32_10(np.arange(512, dtype=np.uint64), 0, 3, philox.S_IDX, k0, k1)
    for n in (1, 5, 20, 31):
        top = (x1.astype(np.uint64) >> np.uint64(32 - n)).astype(np.int64)
        assert np.array_equal(philox.sample_indices(77, 3, 2 ** n, 512), top)


def test_index_uniformity_chi_square():
    # over 1e5 draws from a 100-record ring, per-slot counts uniform within 3 sigma
    idx = np.concatenate([philox.sample_indices(6126, k, 100, 10_000) for k in range(10)])
    counts = np.bincount(idx, minlength=100)
    exp = idx.size / 100
    chi2 = np.sum((counts - exp) ** 2 / exp)
    # chi-square with 99 dof: mean 99, sd sqrt(198) ~ 14.1 -> 3 sigma ~ 141
    assert chi2 < 99 + 3 * np.sqrt(2 * 99)
    z = (counts - exp) / np.sqrt(exp * (1 - 1 / 100))
    assert np.abs(z).max() < 4.5


def test_index_depends_on_seed_step_row():
    a = philox.sample_indices(1, 0, 10**6, 64)
    assert not np.array_equal(a, philox.sample_indices(2, 0, 10**6, 64))
    assert not np.array_equal(a, philox.sample_indices(1, 1, 10**6, 64))
    # rows are addressed by their global id: a shard starting at row0 sees the same values
    assert np.array_equal(philox.sample_indices(1, 0, 10**6, 64)[16:], philox.sample_indices(1, 0, 10**6, 48, row0=16))


def test_uniform_map_exact_endpoints():
    assert philox.uniform_open01(0) == 0.5 * 2.0 ** -23
    assert philox.uniform_open01(0xFFFFFFFF) == 1.0 - 0.5 * 2.0 ** -23
    # representable exactly in float32
    u = philox.uniform_open01(np.arange(0, 2**32, 2**20 + 12345, dtype=np.uint64))
    assert np.array_equal(u.astype(np.float32).astype(np.float64), u)
    assert np.all((u > 0) & (u < 1))


def test_normals_moments_and_independence():
    n = philox.normals(6126, 0, philox.S_EPS, 250_000, 4)
    x = n.ravel()
    N = x.size  # 1e6
    assert abs(x.mean()) < 4 / np.sqrt(N)
    assert abs(x.var() - 1.0) < 4 * np.sqrt(2.0 / N)
    # fourth moment of a standard normal = 3
    assert abs(np.mean(x ** 4) - 3.0) < 4 * np.sqrt(96.0 / N)
    # the cos/sin pair from one block and the two pairs are uncorrelated
    for a, b in ((0, 1), (0, 2), (1, 3), (2, 3)):
        c = np.mean(n[:, a] * n[:, b])
        assert abs(c) < 4 / np.sqrt(n.shape[0])


def test_normals_width_prefix_consistent():
    a = philox.normals(3, 7, philox.S_EPS2, 100, 17)
    b = philox.normals(3, 7, philox.S_EPS2, 100, 6)
    assert np.array_equal(a[:, :6], b)
    assert np.array_equal(philox.normals(3, 7, philox.S_EPS2, 100, 6)[40:],
                          philox.normals(3, 7, philox.S_EPS2, 60, 6, row0=40))
