"""Counter-based sampler identity for the GPU gather kernel.

The reference threads a numpy ``Generator`` through its samplers and calls
``rng.integers(0, n, size)`` (estimators.py:157, :225).  On the GPU each query
owns an independent Philox4x32-10 stream keyed by (seed, query position)
(csrc/sample.cu), so an estimator call needs only a 64-bit seed and the query
position of its first query.  ``PhiloxSampler`` carries both; a numpy
``Generator`` passed as ``rng=`` is converted by drawing one 63-bit seed from
it, so identically seeded generators give identical GPU streams (which is what
makes ``deann(k=0)`` reproduce ``rs_kde`` exactly, test_estimators.py:195-201).
"""

from __future__ import annotations

import numpy as np

__all__ = ["PhiloxSampler", "resolve_sampler"]


class PhiloxSampler:
    """A Philox key plus a running query position.

    Each call consumes ``nq`` query positions, so successive single-query
    calls draw from disjoint streams (like successive ``rng.integers`` calls).
    """

    def __init__(self, seed: int, position: int = 0):
        self.seed = int(seed) & ((1 << 64) - 1)
        self.position = int(position)

    def take(self, nq: int) -> tuple[int, int]:
        base = self.position
        self.position += int(nq)
        return self.seed, base

    def __repr__(self) -> str:
        return f"PhiloxSampler(seed={self.seed:#x}, position={self.position})"


def resolve_sampler(rng) -> PhiloxSampler:
    if isinstance(rng, PhiloxSampler):
        return rng
    if isinstance(rng, (int, np.integer)):
        return PhiloxSampler(int(rng))
    if hasattr(rng, "integers"):
        return PhiloxSampler(int(rng.integers(0, 2**63 - 1)))
    raise TypeError(f"rng must be a numpy Generator, an int seed or a PhiloxSampler, got {type(rng)!r}")
