"""Philox4x32-10 and the random variates the update draws (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading #13 of DESIGN.md: uniform sampling with
replacement over the ring is driven by the counter-based
Philox4x32-10 generator of Salmon et al. (Random123), key = (seed_lo, seed_hi),
counter = (row j, block c, step k, stream S).  Stream ids are fixed below.

Pinned by tests/test_oracle_philox.py against the published Random123 known
answer vectors (tests/golden/philox_kat.txt).
"""

import numpy as np

# Philox4x32 multipliers and Weyl key increments (Random123, philox.h).
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)

# Stream ids (reading #13).
S_IDX, S_EPS, S_EPS2, S_SMOOTH, S_INIT = 1, 2, 3, 4, 5


def _mulhilo(a, b):
    """32x32 -> 64 product split into (hi, lo) 32-bit words."""
    p = np.uint64(a) * b.astype(np.uint64)
    return (p >> np.uint64(32)).astype(np.uint64), (p & _MASK32).astype(np.uint64)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox rounds on counter (c0..c3) with key (k0, k1).

    Arrays (or scalars) of counters broadcast together; returns four uint32
    arrays x0..x3.  One round:  (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by the
    Weyl constants between rounds.
    """
    c0, c1, c2, c3 = np.broadcast_arrays(*[np.asarray(c, dtype=np.uint64) & _MASK32 for c in (c0, c1, c2, c3)])
    c = [c0.copy(), c1.copy(), c2.copy(), c3.copy()]
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + PHILOX_W0) & 0xFFFFFFFF
            k1 = (k1 + PHILOX_W1) & 0xFFFFFFFF
        hi0, lo0 = _mulhilo(PHILOX_M0, c[0])
        hi1, lo1 = _mulhilo(PHILOX_M1, c[2])
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return tuple(x.astype(np.uint32) for x in c)


def key_of(seed):
    """Key = (seed_lo, seed_hi) of a 64-bit seed."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def sample_indices(seed, step, fill, batch, row0=0):
    """Replay indices idx_j = floor((x1*2^32 + x0) * F / 2^64), j = row0..row0+batch-1.

    SURVEY.md §8(a) a1 / reading #13: uniform with replacement over slots
    [0, F).  The 64x64->128 product is evaluated with exact
    Python integers, so this is the definition written out.
    """
    if fill <= 0:
        raise ValueError("fill must be positive")
    k0, k1 = key_of(seed)
    j = np.arange(row0, row0 + batch, dtype=np.uint64)
    x0, x1, _, _ = philox4x32_10(j, 0, step, S_IDX, k0, k1)
    out = np.empty(batch, dtype=np.int64)
    F = int(fill)
    for t in range(batch):
        X = (int(x1[t]) << 32) | int(x0[t])
        out[t] = (X * F) >> 64
    return out


def uniform_open01(x):
    """U(x) = (floor(x / 2^9) + 0.5) * 2^-23, exact in fp32 and fp64 (reading #13 / §8(c) step 2)."""
    x = np.asarray(x, dtype=np.uint64)
    return ((x >> np.uint64(9)).astype(np.float64) + 0.5) * 2.0 ** -23


def normals(seed, step, stream, batch, width, row0=0):
    """Standard normals n[j, q] for rows j = row0.., q = 0..width-1 (§8(c) step 2).

    Block c = q // 4 gives (x0..x3) = Philox(key, (j, c, k, S)); pair
    p = (q mod 4) // 2 uses (x_{2p}, x_{2p+1}); Box-Muller:
    R = sqrt(-2 ln U(x_{2p})), theta = 2 pi U(x_{2p+1}); even q -> R cos theta,
    odd q -> R sin theta.
    """
    k0, k1 = key_of(seed)
    j = np.arange(row0, row0 + batch, dtype=np.uint64)
    out = np.empty((batch, width), dtype=np.float64)
    nblk = (width + 3) // 4
    for c in range(nblk):
        xs = philox4x32_10(j, c, step, stream, k0, k1)
        for p in range(2):
            u1 = uniform_open01(xs[2 * p])
            u2 = uniform_open01(xs[2 * p + 1])
            R = np.sqrt(-2.0 * np.log(u1))
            th = 2.0 * np.pi * u2
            for parity, val in ((0, R * np.cos(th)), (1, R * np.sin(th))):
                q = 4 * c + 2 * p + parity
                if q < width:
                    out[:, q] = val
    return out
