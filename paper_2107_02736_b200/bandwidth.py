"""Bandwidth selection by bracket expansion + geometric bisection on the GPU.

Restates the reference's ``fit_bandwidth`` (analysis.py:256-323, SURVEY §8
row f2): the lower median (analysis.py:201-203) of the exact KDE over a
validation query set is driven to ``target_mu`` within ``rel_tol``.  Every
median evaluation is one batched ``naive_kde`` on the GPU instead of the
reference's cached-distance / blocked-CPU evaluation (analysis.py:224-253),
so configs with 1e6-8e6 rows fit in seconds.  The bracket seed (median
pairwise distance of 100 rows drawn with ``default_rng(0)``) follows
analysis.py:280-294 exactly; that 100x100 seed is control-plane work.
"""

from __future__ import annotations

import math

import numpy as np

from .data import as_gpu_dataset
from .estimators import naive_kde
from .kernels import KernelFamily, KernelSpec

__all__ = ["fit_bandwidth", "NoBandwidthError"]


class NoBandwidthError(RuntimeError):
    """No bandwidth can reach the requested target median KDE (analysis.py:47-55)."""

    def __init__(self, target: float, low: float, high: float):
        self.target = target
        self.achievable = (low, high)
        super().__init__(f"target median KDE {target:g} unreachable; achievable range is [{low:g}, {high:g})")


def _lower_median(values: np.ndarray) -> float:
    ordered = np.sort(values)
    return float(ordered[(len(ordered) - 1) // 2])


def fit_bandwidth(train, validation_queries, kernel_family, target_mu: float, rel_tol: float = 0.01,
                  max_iter: int = 200) -> float:
    family = KernelFamily(getattr(kernel_family, "value", kernel_family))
    if not 0 < target_mu < 1:
        raise ValueError(f"target_mu must be in (0, 1), got {target_mu}")
    queries = np.atleast_2d(np.asarray(validation_queries, dtype=np.float64))
    if queries.shape[0] < 1:
        raise ValueError("validation query set must be nonempty")
    ds = as_gpu_dataset(train)

    def median_kde(h: float) -> float:
        return _lower_median(naive_kde(ds, KernelSpec(family, h), queries).values)

    rng = np.random.default_rng(0)
    picks = rng.choice(ds.n, size=min(100, ds.n), replace=False)
    sample = ds.data[picks].astype(np.float64)
    if family is KernelFamily.LAPLACIAN:
        pair = np.abs(sample[:, None, :] - sample[None, :, :]).sum(axis=2)
    else:
        sq = np.einsum("ij,ij->i", sample, sample)
        pair = np.sqrt(np.maximum(np.add.outer(sq, sq) - 2.0 * (sample @ sample.T), 0.0))
    off_diag = pair[~np.eye(len(sample), dtype=bool)]
    scale = _lower_median(off_diag) if off_diag.size else 1.0
    if scale <= 0.0:
        scale = 1.0

    h_lo = 1e-9 * scale
    med_lo = median_kde(h_lo)
    if abs(med_lo - target_mu) <= rel_tol * target_mu:
        return h_lo
    if med_lo > target_mu:
        raise NoBandwidthError(target_mu, med_lo, 1.0)
    h_hi = scale
    med_hi = median_kde(h_hi)
    doublings = 0
    while med_hi < target_mu and doublings < 64:
        h_lo = h_hi
        h_hi *= 2.0
        med_hi = median_kde(h_hi)
        doublings += 1
    if med_hi < target_mu:
        raise NoBandwidthError(target_mu, med_lo, med_hi)
    for _ in range(max_iter):
        h_mid = math.sqrt(h_lo * h_hi)
        med = median_kde(h_mid)
        if abs(med - target_mu) <= rel_tol * target_mu:
            return h_mid
        if med < target_mu:
            h_lo = h_mid
        else:
            h_hi = h_mid
    raise NoBandwidthError(target_mu, median_kde(h_lo), median_kde(h_hi))
