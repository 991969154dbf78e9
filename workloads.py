"""Seeded synthetic stand-ins for the five BASELINE.json configs.

The paper measures on real datasets that are not in this container
(SURVEY §8(d)); these generators reproduce the SHAPES and
value distributions BASELINE.json prescribes, deterministically from numpy
PCG64 seeds (config index c: cluster centres seed [c, 99], rows seed c, queries seed c+1,
pilot seed c+2;
config 1 uses the reference's own `synth.gaussian_mixture` recipe, restated
here so the GPU box needs no reference checkout).

    c1  n=10,000    d=16   10-cluster mixture, means N(0,4I), sigma=1, h=2.0 fixed
    c2  n=1,000,000 d=128  100-cluster mixture, means N(0,25I), sigma=3, +10, clip [0,255], rint
    c3  n=1,200,000 d=100  200-cluster mixture, means N(0,I), sigma=0.3, rows L2-normalised
    c4  n=60,000    d=784  each coordinate 0 w.p. 0.8 else U(0,1]
    c5  n=8,000,000 d=96   1000 clusters, means N(0,16I), sigma=1, Dirichlet(1) weights

Bandwidths for c2-c5 follow the reference's median-1e-3 bisection rule
(analysis.fit_bandwidth semantics), evaluated on the GPU over the 1,000-query
pilot set (paper_2107_02736_b200.fit_bandwidth).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Workload", "make", "CONFIGS"]


@dataclass
class Workload:
    name: str
    X: np.ndarray          # (n, d) float32
    Q: np.ndarray          # (nq, d) float64
    pilot: np.ndarray | None
    family: str
    h: float | None        # fixed bandwidth (None -> median-1e-3 bisection)
    k: int
    m: int


def _normal32(rng, shape, scale=1.0):
    out = rng.standard_normal(shape, dtype=np.float32)
    if scale != 1.0:
        out *= np.float32(scale)
    return out


def _c1(nq=1000, n=10_000):
    # synth.gaussian_mixture(10_000, 16, 10, seed=0, center_scale=2.0, component_std=1.0) (synth.py:18-37)
    rng = np.random.default_rng(0)
    centers = rng.normal(0.0, 2.0, size=(10, 16))
    labels = np.arange(n) % 10
    X = (centers[labels] + rng.normal(0.0, 1.0, size=(n, 16))).astype(np.float32)
    # synth.mixture_queries(0, 1000, 16, 10, 2.0, 1.0) (synth.py:40-58, query seed 1)
    qrng = np.random.default_rng(1)
    ql = qrng.integers(0, 10, size=nq)
    Q = centers[ql] + qrng.normal(0.0, 1.0, size=(nq, 16))
    return Workload("c1", X, Q, None, "gaussian", 2.0, 50, 500)


def _c2_rows(seed, n):
    d = 128
    crng = np.random.default_rng([2, 99])
    centers = crng.normal(0.0, 5.0, size=(100, d)).astype(np.float32)
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 100, size=n)
    out = np.empty((n, d), dtype=np.float32)
    step = 1 << 18
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        blk = centers[labels[lo:hi]] + _normal32(rng, (hi - lo, d), 3.0)
        blk += np.float32(10.0)
        np.clip(blk, 0.0, 255.0, out=blk)
        np.rint(blk, out=blk)
        out[lo:hi] = blk
    return out


def _c2(n=1_000_000, nq=10_000):
    X = _c2_rows(2, n)
    Q = _c2_rows(3, nq).astype(np.float64)
    P = _c2_rows(4, 1000).astype(np.float64)
    return Workload("c2", X, Q, P, "gaussian", None, 100, 1000)


def _c3_rows(seed, n):
    d = 100
    crng = np.random.default_rng([3, 99])
    centers = crng.normal(0.0, 1.0, size=(200, d)).astype(np.float32)
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 200, size=n)
    out = np.empty((n, d), dtype=np.float32)
    step = 1 << 18
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        blk = centers[labels[lo:hi]] + _normal32(rng, (hi - lo, d), 0.3)
        blk /= np.linalg.norm(blk, axis=1, keepdims=True)
        out[lo:hi] = blk
    return out


def _c3(n=1_200_000, nq=10_000):
    return Workload("c3", _c3_rows(3, n), _c3_rows(4, nq).astype(np.float64), _c3_rows(5, 1000).astype(np.float64),
                    "gaussian", None, 100, 1000)


def _c4_rows(seed, n):
    rng = np.random.default_rng(seed)
    d = 784
    out = np.empty((n, d), dtype=np.float32)
    step = 1 << 14
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        keep = rng.random((hi - lo, d), dtype=np.float32) >= np.float32(0.8)
        val = np.float32(1.0) - rng.random((hi - lo, d), dtype=np.float32)  # U(0, 1]
        out[lo:hi] = np.where(keep, val, np.float32(0.0))
    return out


def _c4(n=60_000, nq=10_000, family="exponential"):
    return Workload("c4", _c4_rows(4, n), _c4_rows(5, nq).astype(np.float64), _c4_rows(6, 1000).astype(np.float64),
                    family, None, 50, 500)


def _c5_rows(seed, n):
    d = 96
    crng = np.random.default_rng([5, 99])
    centers = crng.normal(0.0, 4.0, size=(1000, d)).astype(np.float32)
    weights = crng.dirichlet(np.ones(1000))
    rng = np.random.default_rng(seed)
    labels = rng.choice(1000, size=n, p=weights)
    out = np.empty((n, d), dtype=np.float32)
    step = 1 << 18
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        out[lo:hi] = centers[labels[lo:hi]] + _normal32(rng, (hi - lo, d), 1.0)
    return out


def _c5(n=8_000_000, nq=100_000):
    return Workload("c5", _c5_rows(5, n), _c5_rows(6, nq).astype(np.float64), _c5_rows(7, 1000).astype(np.float64),
                    "gaussian", None, 100, 2000)


CONFIGS = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4, "c5": _c5}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
