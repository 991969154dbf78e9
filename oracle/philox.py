"""NumPy Philox4x32-10 stream of the GPU sampler — TEST INFRASTRUCTURE ONLY.

Restates csrc/sample.cu's draw rule so the oracle can replay the GPU's
sample stream through the reference's `rng.integers` protocol
(estimators.py:157, :225):

    r = philox4x32_10(ctr = {t_lo, t_hi, j_lo, j_hi}, key = {seed_lo, seed_hi})
    row_t = floor(((r1 << 32) | r0) * N / 2^64)

Philox4x32-10 follows Salmon et al., "Parallel random numbers: as easy as
1, 2, 3" (SC'11): round multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key
increments 0x9E3779B9 / 0xBB67AE85, key bumped before rounds 2..10.
The implementation is checked against the published Random123 known-answer
vectors in tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key: tuple[int, int]) -> np.ndarray:
    """ctr: (N, 4) uint32-valued array; returns (N, 4) uint64 (values < 2^32)."""
    c = np.asarray(ctr, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = c[:, 0].copy(), c[:, 1].copy(), c[:, 2].copy(), c[:, 3].copy()
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = c0 * M0
        p1 = c2 * M1
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
    return np.stack([c0, c1, c2, c3], axis=1)


def _mulhi64(a: np.ndarray, n: int) -> np.ndarray:
    """floor(a * n / 2^64) for uint64 a and n < 2^63, exact via 32-bit limbs."""
    a = a.astype(np.uint64)
    a_lo, a_hi = a & MASK32, a >> np.uint64(32)
    n_lo, n_hi = np.uint64(n & 0xFFFFFFFF), np.uint64(n >> 32)
    ll = a_lo * n_lo
    lh = a_lo * n_hi
    hl = a_hi * n_lo
    hh = a_hi * n_hi
    mid = (ll >> np.uint64(32)) + (lh & MASK32) + (hl & MASK32)
    return hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))


def draws(seed: int, query_pos: int, t0: int, count: int, n: int) -> np.ndarray:
    """Rows of draws t0 .. t0+count-1 of query position `query_pos`."""
    t = np.arange(t0, t0 + count, dtype=np.uint64)
    j = np.uint64(query_pos)
    ctr = np.stack([t & MASK32, t >> np.uint64(32), np.full_like(t, j & MASK32), np.full_like(t, j >> np.uint64(32))],
                   axis=1)
    r = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    v = (r[:, 1] << np.uint64(32)) | r[:, 0]
    return _mulhi64(v, int(n)).astype(np.int64)


class IndexReplay:
    """Duck-typed rng: `.integers(0, n, size)` returns the next entries of one
    query's Philox stream (SURVEY §8(c) IndexReplay shim)."""

    def __init__(self, seed: int, query_pos: int, n: int):
        self.seed, self.query_pos, self.n, self.t = int(seed), int(query_pos), int(n), 0

    def integers(self, low, high, size=None):
        if low != 0 or high != self.n:
            raise ValueError(f"replay stream is over [0, {self.n}), asked [{low}, {high})")
        count = 1 if size is None else int(size)
        out = draws(self.seed, self.query_pos, self.t, count, self.n)
        self.t += count
        return out if size is not None else int(out[0])


class NeighborReplay:
    """Duck-typed AnnIndex replaying fixed neighbours (cf. test_acceptance.py:60-68)."""

    def __init__(self, indices, sq_distances):
        self.indices = np.asarray(indices, dtype=np.int64)
        self.sq_distances = np.asarray(sq_distances, dtype=np.float64)

    def __call__(self, y, k):
        return self.indices[:k], self.sq_distances[:k]
