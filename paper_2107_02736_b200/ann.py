"""Neighbour layer: the exact brute-force index on the GPU.

Mirrors reference ann.py:49-121.  ``GpuBruteForceIndex`` is an ``AnnIndex``
(query(y, k) -> NeighborList) whose search is the tensor-core distance sweep
+ certified exact re-rank of ``dk_knn`` (csrc/knn.cu): identical neighbour
sets and (d2, idx) order as ``brute_force_knn`` (ties to the lower index,
ann.py:82-102), with fp64 squared distances by direct difference (within the
reference's 1e-6 recomputation contract, test_ann.py:181-188).
"""

from __future__ import annotations

import abc
from dataclasses import dataclass

import numpy as np

from . import _lib
from .data import as_gpu_dataset

__all__ = ["NeighborList", "AnnIndex", "GpuBruteForceIndex", "BruteForceIndex", "brute_force_knn"]


@dataclass
class NeighborList:
    """Distinct row indices with nondecreasing squared distances (ann.py:49-67)."""

    indices: np.ndarray
    sq_distances: np.ndarray

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.int64)
        self.sq_distances = np.asarray(self.sq_distances, dtype=np.float64)
        if self.indices.shape != self.sq_distances.shape:
            raise ValueError("indices and sq_distances must have equal length")
        if len(np.unique(self.indices)) != len(self.indices):
            raise ValueError("neighbor indices must be distinct")
        if len(self.sq_distances) > 1 and np.any(np.diff(self.sq_distances) < 0):
            raise ValueError("sq_distances must be nondecreasing")

    def __len__(self) -> int:
        return len(self.indices)


class AnnIndex(abc.ABC):
    """Black-box k-NN interface (ann.py:70-75)."""

    @abc.abstractmethod
    def query(self, query, k: int) -> NeighborList:
        """Return up to k near neighbours of `query`."""


def _queries64(queries, d: int) -> np.ndarray:
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
    if q.shape[1] != d:
        raise ValueError(f"dimension mismatch: queries d={q.shape[1]}, dataset d={d}")
    return q


def knn_batch(dataset, queries, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Exact k-NN of every query row: (indices (nq, k) int64, sq_distances (nq, k) fp64)."""
    ds = as_gpu_dataset(dataset)
    if not 1 <= k <= ds.n:
        raise ValueError(f"k={k} out of range [1, {ds.n}]")
    q = _queries64(queries, ds.d)
    idx = _lib.host_empty((q.shape[0], k), np.int64)
    d2 = _lib.host_empty((q.shape[0], k), np.float64)
    _lib.check(_lib.load().dk_knn(ds.handle, q.ctypes.data, q.shape[0], k, idx.ctypes.data, d2.ctypes.data,
                                  _lib.current_stream()))
    return idx, d2


def brute_force_knn(dataset, query, k: int) -> NeighborList:
    """Exact k nearest rows by squared L2 distance (ann.py:105-111)."""
    ds = as_gpu_dataset(dataset)
    if not 1 <= k <= ds.n:
        raise ValueError(f"k={k} out of range [1, {ds.n}]")
    idx, d2 = knn_batch(ds, np.asarray(query, dtype=np.float64).reshape(1, -1), k)
    return NeighborList(indices=idx[0], sq_distances=d2[0])


class GpuBruteForceIndex(AnnIndex):
    """Exact brute force on the GPU; drop-in for ``BruteForceIndex`` (ann.py:114-121)."""

    def __init__(self, dataset):
        self.dataset = as_gpu_dataset(dataset)

    def query(self, query, k: int) -> NeighborList:
        return brute_force_knn(self.dataset, query, k)

    def query_batch(self, queries, k: int) -> tuple[np.ndarray, np.ndarray]:
        return knn_batch(self.dataset, queries, k)


BruteForceIndex = GpuBruteForceIndex
