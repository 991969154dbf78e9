"""KDE estimators on the GPU — drop-in for reference estimators.py.

Same names, signatures, return types and ValueError preconditions as
``naive_kde`` (estimators.py:122-149), ``rs_kde`` (:152-164), ``deann``
(:306-379) and ``deann_batch`` (:382-410).  The arithmetic runs in the CUDA
kernels behind the C-ABI:

* naive_kde  -> dk_naive: fused tcgen05 distance tile + exp + row sum
  (gaussian/exponential) or the CUDA-core L1 kernel (laplacian);
* rs_kde     -> dk_sample without exclusions (Philox-indexed gather);
* deann      -> dk_deann (exact k-NN + exclusion sampling + combine) when the
  index is the GPU brute force; any other AnnIndex is queried as a black box
  and its neighbours drive dk_sample / dk_eval_rows / dk_kernel_values;
* rsp_kde / deann(rsp_state=) -> dk_rsp_walk: the permuted sampler streams
  contiguous windows of the device-resident permuted rows (rsp.cu), with the
  reference's cursor semantics (shared threading or independent cursors).

Difference to the reference, by design: the uniform sampler is a
counter-based Philox stream per query (sampler.py) instead of numpy's PCG64.
The permuted sampler is deterministic and matches the reference exactly
(same PCG64 permutation, same cursor arithmetic).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .ann import GpuBruteForceIndex
from .data import Dataset, PermutedDataset, as_gpu_dataset, as_gpu_permuted, permute
from .kernels import KernelFamily, as_spec
from .sampler import resolve_sampler

__all__ = [
    "Estimate", "BatchKde", "RspState", "naive_kde", "rs_kde", "rsp_kde", "deann", "deann_batch",
    "naive_kde_into", "deann_arrays", "kernel_from_distance", "EstimateList",
]


@dataclass(slots=True)
class Estimate:
    """A single KDE estimate plus its cost counters (estimators.py:57-72)."""

    value: float
    kernel_evals: int
    neighbors_used: int
    samples_used: int
    truncated: bool = False
    clamped: bool = False


@dataclass
class BatchKde:
    """Exact KDE values for a query batch plus the total kernel-eval count (estimators.py:75-80)."""

    values: np.ndarray
    kernel_evals: int


class EstimateList(list):
    """``list[Estimate]`` of a batch, built from the batch's result arrays on first use.

    ``deann_batch`` returns one ``Estimate`` per query (estimators.py:382-410).  Creating
    10,000 Python objects costs about as much host time as the whole device batch, so the
    list keeps the value / counter arrays and materialises the ``Estimate`` objects the first
    time it is read (indexing, iteration, len, comparison, copy, mutation, pickling...).
    After that it is an ordinary list.  ``values`` / ``kernel_evals`` / ... give the arrays
    without materialising.
    """

    __slots__ = ("values", "kernel_evals", "neighbors_used", "samples_used", "truncated", "clamped", "_lazy")

    def __init__(self, values, kernel_evals, neighbors_used, samples_used, truncated=False, clamped=False):
        super().__init__()
        n = len(values)
        self.values = np.asarray(values, dtype=np.float64)
        self.kernel_evals = np.broadcast_to(np.asarray(kernel_evals, dtype=np.int64), (n,))
        self.neighbors_used = np.broadcast_to(np.asarray(neighbors_used, dtype=np.int64), (n,))
        self.samples_used = np.broadcast_to(np.asarray(samples_used, dtype=np.int64), (n,))
        self.truncated = np.broadcast_to(np.asarray(truncated, dtype=bool), (n,))
        self.clamped = np.broadcast_to(np.asarray(clamped, dtype=bool), (n,))
        self._lazy = True

    def _m(self):
        if self._lazy:
            self._lazy = False
            list.extend(self, map(Estimate, self.values.tolist(), self.kernel_evals.tolist(),
                                  self.neighbors_used.tolist(), self.samples_used.tolist(), self.truncated.tolist(),
                                  self.clamped.tolist()))
        return self

    def __len__(self):
        return len(self.values) if self._lazy else list.__len__(self)

    def __bool__(self):
        return len(self) > 0

    def __array__(self, dtype=None, copy=None):
        return np.asarray(list(self._m()), dtype=dtype if dtype is not None else object)

    def __reduce_ex__(self, protocol):
        return (list, (list(self._m()),))


def _lazy_method(name):
    base = getattr(list, name)

    def method(self, *args, **kwargs):
        return base(self._m(), *args, **kwargs)

    method.__name__ = name
    return method


for _name in ("__getitem__", "__iter__", "__contains__", "__reversed__", "__repr__", "__eq__", "__ne__", "__lt__",
              "__le__", "__gt__", "__ge__", "__add__", "__mul__", "__rmul__", "__iadd__", "__imul__", "__setitem__",
              "__delitem__", "__sizeof__", "append", "extend", "insert", "pop", "remove", "clear", "index", "count",
              "copy", "sort", "reverse"):
    setattr(EstimateList, _name, _lazy_method(_name))
EstimateList.__radd__ = lambda self, other: list(other) + list(self._m())  # noqa: E731
EstimateList.__hash__ = None


def _queries64(queries, d: int) -> np.ndarray:
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.float64)))
    if q.shape[1] != d:
        raise ValueError(f"dimension mismatch: queries d={q.shape[1]}, dataset d={d}")
    return q


def _query64(query, d: int) -> np.ndarray:
    y = np.ascontiguousarray(np.asarray(query, dtype=np.float64).ravel())
    if y.shape[0] != d:
        raise ValueError(f"dimension mismatch: query d={y.shape[0]}, dataset d={d}")
    return y


# ---------------------------------------------------------------- exact


def naive_kde_into(dataset: Dataset, kernel, queries, out, *, sums: bool = False, stream=None) -> None:
    """Exact KDE into a caller buffer.  ``queries`` (nq, d) fp64 and ``out`` (nq,)
    fp64 may be numpy arrays or torch CUDA tensors (device buffers skip all copies)."""
    spec = as_spec(kernel)
    nq = int(queries.shape[0])
    _lib.check(_lib.load().dk_naive(dataset.handle, _lib.ptr(queries), nq, _lib.family_code(spec.family),
                                    spec.bandwidth, _lib.DK_OUT_SUM if sums else 0, _lib.ptr(out),
                                    stream if stream is not None else _lib.current_stream()))


def naive_kde(dataset, kernel, queries) -> BatchKde:
    """Exact KDE of every query against the full dataset (estimators.py:122-149)."""
    ds = as_gpu_dataset(dataset)
    spec = as_spec(kernel)
    q = _queries64(queries, ds.d)
    values = np.empty(q.shape[0], dtype=np.float64)
    naive_kde_into(ds, spec, q, values)
    return BatchKde(values=values, kernel_evals=q.shape[0] * ds.n)


def kernel_from_distance(spec, dist):
    """Kernel values from precomputed family distances (kernels.py:65-83), on the GPU."""
    spec = as_spec(spec)
    scalar = np.isscalar(dist) or np.ndim(dist) == 0
    d = np.ascontiguousarray(np.asarray(dist, dtype=np.float64).ravel())
    if not np.all(np.isfinite(d)):
        raise ValueError("distance must be finite")
    if np.any(d < 0.0):
        raise ValueError("distance must be nonnegative")
    out = np.empty_like(d)
    if d.size:
        _lib.check(_lib.load().dk_kernel_values(_lib.family_code(spec.family), spec.bandwidth, d.ctypes.data,
                                                d.size, out.ctypes.data, None))
    if scalar:
        return float(out[0])
    return out.reshape(np.shape(dist))


def kernel_pair(spec, x, y) -> float:
    """Kernel value between two points with the family's own metric (kernels.py:86-106)."""
    spec = as_spec(spec)
    xv = np.asarray(x, dtype=np.float64).ravel()
    yv = np.asarray(y, dtype=np.float64).ravel()
    if xv.shape != yv.shape:
        raise ValueError(f"dimension mismatch: {xv.shape[0]} vs {yv.shape[0]}")
    if xv.size == 0:
        raise ValueError("vectors must have dimension >= 1")
    diff = xv - yv
    if spec.family is KernelFamily.GAUSSIAN:
        dist = float(diff @ diff)
    elif spec.family is KernelFamily.EXPONENTIAL:
        dist = math.sqrt(float(diff @ diff))
    else:
        dist = float(np.abs(diff).sum())
    return kernel_from_distance(spec, dist)


def dataset_sha256(dataset) -> str:
    """SHA-256 of the rows as little-endian fp32 (harness.py:183-184)."""
    data = getattr(dataset, "data", dataset)
    return hashlib.sha256(np.ascontiguousarray(data, dtype="<f4").tobytes()).hexdigest()


def ground_truth(dataset, queries, kernel) -> dict:
    """Exact KDE values plus a manifest tying them to their inputs (harness.py:187-196), on the GPU."""
    spec = as_spec(kernel)
    values = naive_kde(dataset, spec, queries).values
    return {
        "kernel": spec.family.value,
        "bandwidth": spec.bandwidth,
        "dataset_sha256": dataset_sha256(dataset),
        "n_queries": int(len(values)),
        "values": [float(v) for v in values],
    }


# ---------------------------------------------------------------- sampling


def _sample_sums(ds: Dataset, spec, q: np.ndarray, m: int, seed: int, base: int, excl=None, excl_cnt=None,
                 stride: int = 0, export: bool = False):
    nq = q.shape[0]
    z = np.empty(nq, dtype=np.float64)
    acc = _lib.host_empty((nq, m), np.int64) if export else None
    _lib.check(_lib.load().dk_sample(ds.handle, q.ctypes.data, nq, _lib.family_code(spec.family), spec.bandwidth,
                                     m, seed, base, _lib.ptr(excl), _lib.ptr(excl_cnt), stride, z.ctypes.data,
                                     _lib.ptr(acc), None, None))
    return z, acc


def rs_kde(dataset, kernel, query, m: int, rng) -> Estimate:
    """Uniform sampling with replacement: mean kernel value over m draws (estimators.py:152-164)."""
    if m < 1:
        raise ValueError(f"m={m} must be >= 1")
    ds = as_gpu_dataset(dataset)
    spec = as_spec(kernel)
    y = _query64(query, ds.d).reshape(1, -1)
    seed, base = resolve_sampler(rng).take(1)
    z, _ = _sample_sums(ds, spec, y, m, seed, base)
    return Estimate(value=float(z[0] / m), kernel_evals=m, neighbors_used=0, samples_used=m)


# ---------------------------------------------------------------- permuted sampler


@dataclass
class RspState:
    """Permuted copy of the data plus the running cursor (estimators.py:83-96)."""

    permuted: PermutedDataset
    cursor: int = 0

    @classmethod
    def from_dataset(cls, dataset, seed: int, cursor: int = 0) -> "RspState":
        return cls(permuted=permute(dataset, seed), cursor=cursor)

    @property
    def n(self) -> int:
        return self.permuted.n


def _rsp_walk(state, spec, q: np.ndarray, m: int, excl, independent: bool):
    """One dk_rsp_walk over a query batch; updates the shared cursor (unless independent)."""
    pds = as_gpu_permuted(state.permuted)
    nq = q.shape[0]
    z = np.empty(nq, dtype=np.float64)
    taken = np.empty(nq, dtype=np.int32)
    cur = ctypes.c_int64()
    ex = None if excl is None else np.ascontiguousarray(excl, dtype=np.int64)
    _lib.check(_lib.load().dk_rsp_walk(pds.base.handle, q.ctypes.data, nq, _lib.family_code(spec.family),
                                       spec.bandwidth, m, _lib.ptr(ex), 0 if ex is None else ex.shape[1],
                                       int(state.cursor), 1 if independent else 0, z.ctypes.data, taken.ctypes.data,
                                       ctypes.byref(cur), _lib.current_stream()))
    if not independent:
        state.cursor = int(cur.value)
    return z, taken


def rsp_kde(state, kernel, query, m: int) -> Estimate:
    """Permuted contiguous sampling: mean over the next m permuted rows, cursor += m (estimators.py:180-200)."""
    n = state.n
    if not 1 <= m <= n:
        raise ValueError(f"m={m} out of range [1, {n}]")
    spec = as_spec(kernel)
    pds = as_gpu_permuted(state.permuted)
    y = _query64(query, pds.base.d).reshape(1, -1)
    z, _ = _rsp_walk(state, spec, y, m, None, False)
    return Estimate(value=float(z[0] / m), kernel_evals=m, neighbors_used=0, samples_used=m)


def _z1_from_neighbors(ds: Dataset, spec, q: np.ndarray, idx: np.ndarray, d2: np.ndarray) -> np.ndarray:
    """Z1 per query: kernel of the exact neighbour distances (L2 families, estimators.py:349-351)
    or re-evaluated L1 (laplacian, :346-348), on the device."""
    nq, k = idx.shape
    if spec.family is KernelFamily.LAPLACIAN:
        out = np.empty(nq, dtype=np.float64)
        r = np.ascontiguousarray(idx, dtype=np.int64)
        _lib.check(_lib.load().dk_eval_rows(ds.handle, q.ctypes.data, nq, _lib.DK_LAPLACIAN, spec.bandwidth,
                                            r.ctypes.data, None, k, out.ctypes.data, None))
        return out / k
    dist = d2 if spec.family is KernelFamily.GAUSSIAN else np.sqrt(d2)
    return kernel_from_distance(spec, dist).reshape(nq, k).mean(axis=1)


# ---------------------------------------------------------------- DEANN


def _validate(n: int, d: int, k: int, m: int, rng, rsp_state):
    # estimators.py:322-335, same order and messages
    if not 0 <= k <= n:
        raise ValueError(f"k={k} out of range [0, {n}]")
    if m < 0:
        raise ValueError(f"m={m} must be >= 0")
    if m > 0 and k >= n:
        raise ValueError("m > 0 requires k + 1 <= n so the remainder is nonempty")
    if m > 0 and (rng is None) == (rsp_state is None):
        raise ValueError("give exactly one of rng= or rsp_state= when m > 0")
    if rsp_state is not None and rsp_state.n != n:
        raise ValueError("rsp_state was built for a different dataset size")


def _is_gpu_bruteforce(ann, ds: Dataset) -> bool:
    if isinstance(ann, GpuBruteForceIndex):
        return ann.dataset is ds
    # the reference's own BruteForceIndex over the same rows is also exact brute force
    cls = type(ann)
    if cls.__name__ == "BruteForceIndex" and hasattr(ann, "dataset"):
        try:
            return as_gpu_dataset(ann.dataset) is ds
        except TypeError:
            return False
    return False


def deann_arrays(dataset, kernel, queries, k: int, m: int, *, seed: int, query_base: int = 0,
                 export_neighbors: bool = False, export_samples: bool = False):
    """Batch DEANN with exact GPU brute force + Philox sampling.

    Returns (values (nq,), neighbor_idx (nq, k) or None, sample_idx (nq, m) or None).
    """
    ds = as_gpu_dataset(dataset)
    spec = as_spec(kernel)
    q = _queries64(queries, ds.d)
    nq = q.shape[0]
    values = np.empty(nq, dtype=np.float64)
    nbr = _lib.host_empty((nq, k), np.int64) if (export_neighbors and k > 0) else None
    smp = _lib.host_empty((nq, m), np.int64) if (export_samples and m > 0) else None
    _lib.check(_lib.load().dk_deann(ds.handle, q.ctypes.data, nq, _lib.family_code(spec.family), spec.bandwidth,
                                    k, m, int(seed), int(query_base), values.ctypes.data, _lib.ptr(nbr), None,
                                    _lib.ptr(smp), _lib.current_stream()))
    return values, nbr, smp


def deann(dataset, kernel, ann, query, k: int, m: int, *, rng=None, rsp_state=None) -> Estimate:
    """Combined estimator: exact near part from the index, sampled far part (estimators.py:306-379)."""
    ds = as_gpu_dataset(dataset)
    spec = as_spec(kernel)
    n = ds.n
    _validate(n, ds.d, k, m, rng, rsp_state)
    y = _query64(query, ds.d)
    if rsp_state is not None and m > 0:
        return _deann_rsp(ds, spec, ann, y.reshape(1, -1), k, m, rsp_state, False)[0]
    seed, base = resolve_sampler(rng).take(1) if (m > 0) else (0, 0)
    if k == 0 or _is_gpu_bruteforce(ann, ds):
        values, _, _ = deann_arrays(ds, spec, y.reshape(1, -1), k, m, seed=seed, query_base=base)
        k_hat = k
        return Estimate(value=float(values[0]), kernel_evals=k_hat + m, neighbors_used=k_hat, samples_used=m,
                        truncated=(m == 0 and k_hat < n))
    # black-box index: neighbours from `ann`, everything else on the GPU
    neighbors = ann.query(y, k)
    x1 = np.ascontiguousarray(np.asarray(neighbors.indices, dtype=np.int64))
    k_hat = len(x1)
    if k_hat == 0:
        z1 = 0.0
    elif spec.family is KernelFamily.LAPLACIAN:
        out = np.empty(1, dtype=np.float64)
        _lib.check(_lib.load().dk_eval_rows(ds.handle, y.ctypes.data, 1, _lib.DK_LAPLACIAN, spec.bandwidth,
                                            x1.ctypes.data, None, k_hat, out.ctypes.data, None))
        z1 = float(out[0] / k_hat)
    else:
        d2 = np.asarray(neighbors.sq_distances, dtype=np.float64)
        dist = d2 if spec.family is KernelFamily.GAUSSIAN else np.sqrt(d2)
        z1 = float(np.mean(kernel_from_distance(spec, dist)))
    if m == 0:
        return Estimate(value=(k_hat / n) * z1, kernel_evals=k_hat, neighbors_used=k_hat, samples_used=0,
                        truncated=k_hat < n)
    excl = x1.reshape(1, -1) if k_hat else None
    z, _ = _sample_sums(ds, spec, y.reshape(1, -1), m, seed, base, excl=excl, stride=max(k_hat, 1))
    z2 = float(z[0] / m)
    value = (k_hat / n) * z1 + ((n - k_hat) / n) * z2
    return Estimate(value=value, kernel_evals=k_hat + m, neighbors_used=k_hat, samples_used=m)


def deann_batch(dataset, kernel, ann, queries, k: int, m: int, *, rng=None, rsp_state=None,
                independent_cursors: bool = False) -> list[Estimate]:
    """Evaluate a query batch (estimators.py:382-410); one fused GPU call for brute force."""
    ds = as_gpu_dataset(dataset)
    spec = as_spec(kernel)
    q = _queries64(queries, ds.d)
    n = ds.n
    _validate(n, ds.d, k, m, rng, rsp_state)
    if rsp_state is not None and m > 0:
        return _deann_rsp(ds, spec, ann, q, k, m, rsp_state, independent_cursors)
    if k == 0 or _is_gpu_bruteforce(ann, ds):
        seed, base = resolve_sampler(rng).take(q.shape[0]) if m > 0 else (0, 0)
        values, _, _ = deann_arrays(ds, spec, q, k, m, seed=seed, query_base=base)
        return EstimateList(values, k + m, k, m, truncated=(m == 0 and k < n))
    if _is_gpu_ivf(ann, ds):
        return _deann_ivf_batch(ds, spec, ann, q, k, m, rng)
    # black-box index: one call per query in query order (estimators.py:405-409) over ONE
    # sampler, so query j draws from stream position base + j exactly as the fused batch does
    # (an int seed must not restart the stream at every query)
    sampler = resolve_sampler(rng) if m > 0 else None
    return [deann(ds, spec, ann, q[j], k, m, rng=sampler) for j in range(q.shape[0])]


def _is_gpu_ivf(ann, ds: Dataset) -> bool:
    from .ivf import IvfAnnIndex

    return isinstance(ann, IvfAnnIndex) and ann._ds is ds


def _deann_ivf_batch(ds: Dataset, spec, ann, q: np.ndarray, k: int, m: int, rng) -> list[Estimate]:
    """DEANN over a batch with the GPU IVF index, in one device call (dk_deann_ivf): one
    probed query pass for all queries, neighbour lists of per-query length k_hat (ann.py:30-31:
    a short probe set is not an error), Z1 from their distances, then one Philox sampling
    pass excluding each query's list (estimators.py:338-372)."""
    n = ds.n
    nq = q.shape[0]
    values = np.empty(nq, dtype=np.float64)
    khat = np.empty(nq, dtype=np.int32)
    seed, base = resolve_sampler(rng).take(nq) if m > 0 else (0, 0)
    _lib.check(_lib.load().dk_deann_ivf(ann._dev.handle, q.ctypes.data, nq, _lib.family_code(spec.family),
                                        spec.bandwidth, k, m, ann.n_probe, seed, base, values.ctypes.data,
                                        khat.ctypes.data, _lib.current_stream()))
    if m == 0:
        return EstimateList(values, khat, khat, 0, truncated=khat < n)
    return EstimateList(values, khat.astype(np.int64) + m, khat, m)


def _deann_rsp(ds: Dataset, spec, ann, q: np.ndarray, k: int, m: int, state, independent: bool) -> list[Estimate]:
    """DEANN with the permuted sampler over a query batch (DEANNP; estimators.py:306-379, 249-303, 394-409)."""
    n = ds.n
    nq = q.shape[0]
    if k > 0 and _is_gpu_bruteforce(ann, ds):
        from .ann import knn_batch

        idx, d2 = knn_batch(ds, q, k)
        z1 = _z1_from_neighbors(ds, spec, q, idx, d2)
        k_hat = np.full(nq, k)
    elif k > 0:  # black-box index: one query at a time, lists may be shorter than k
        if nq != 1:
            return [_deann_rsp(ds, spec, ann, q[j:j + 1], k, m, state, False)[0] if not independent else
                    _deann_rsp_indep(ds, spec, ann, q, j, k, m, state) for j in range(nq)]
        nb = ann.query(q[0], k)
        x1 = np.asarray(nb.indices, dtype=np.int64)
        if len(x1) == 0:
            return _deann_rsp(ds, spec, None, q, 0, m, state, independent)
        idx = x1.reshape(1, -1)
        d2 = np.asarray(nb.sq_distances, dtype=np.float64).reshape(1, -1)
        z1 = _z1_from_neighbors(ds, spec, q, idx, d2)
        k_hat = np.full(1, len(x1))
    else:
        idx, z1, k_hat = None, np.zeros(nq), np.zeros(nq, dtype=np.int64)
    z, taken = _rsp_walk(state, spec, q, m, idx, independent)
    kh = np.asarray(k_hat, dtype=np.int64)
    t = taken.astype(np.int64)
    z2 = np.divide(z, t, out=np.zeros_like(z), where=t > 0)
    value = (kh / n) * np.asarray(z1, dtype=np.float64) + ((n - kh) / n) * z2
    return EstimateList(value, kh + t, kh, t, clamped=t < m)


def _deann_rsp_indep(ds, spec, ann, q, j, k, m, state):
    sub = RspState(permuted=as_gpu_permuted(state.permuted), cursor=(j * state.n) // q.shape[0])
    return _deann_rsp(ds, spec, ann, q[j:j + 1], k, m, sub, False)[0]
