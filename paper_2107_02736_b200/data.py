"""GPU-resident dataset: the "fit" of every estimator.

Mirrors reference ``Dataset`` (data.py:45-87): an immutable row-major n x d
float32 matrix with fp64 squared row norms.  ``Dataset.from_array`` uploads
the rows once through ``dk_fit`` (finiteness check, fp64 norms and the
tensor-core operand encodings are all computed on the device), after which
every estimator call only moves queries and results.

Any object with a ``.data`` float32 (n, d) array — e.g. the reference's own
``deann.Dataset`` — is accepted by the estimators and fitted on first use
(cached per object).
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib

__all__ = ["Dataset", "as_gpu_dataset", "PermutedDataset", "permute", "as_gpu_permuted"]

_PRECISION = {"auto": _lib.DK_PREC_AUTO, "split3": _lib.DK_PREC_SPLIT3, "fp16": _lib.DK_PREC_FP16}


class Dataset:
    """Immutable rows on the host (``data``) plus a fitted device handle."""

    def __init__(self, data: np.ndarray, handle, *, device: int, global_offset: int, global_n: int,
                 precision: str):
        self.data = data
        self._handle = handle
        self.device = device
        self.global_offset = global_offset
        self.global_n = global_n
        self.precision = precision
        self._sq_norms = None
        self._finalizer = weakref.finalize(self, _free_handle, handle)

    @classmethod
    def from_array(cls, arr, *, device: int = 0, precision: str = "auto", global_offset: int = 0,
                   global_n: int | None = None) -> "Dataset":
        """Validate and upload rows (reference Dataset.from_array, data.py:53-67).

        ``global_offset``/``global_n`` describe this array as one row shard of a
        larger dataset (dataset-sharded multi-GPU mode, see sharded.py).
        """
        data = np.ascontiguousarray(arr, dtype=np.float32)
        if data.ndim != 2:
            raise ValueError(f"dataset must be 2-dimensional, got shape {data.shape}")
        n, d = data.shape
        if n < 1 or d < 1:
            raise ValueError(f"dataset must have n >= 1 and d >= 1, got {n} x {d}")
        if precision not in _PRECISION:
            raise ValueError(f"precision must be one of {sorted(_PRECISION)}, got {precision!r}")
        lib = _lib.load()
        opts = _lib.FitOpts(device, _PRECISION[precision], int(global_offset), int(global_n or 0))
        h = ctypes.c_void_p()
        _lib.check(lib.dk_fit(data.ctypes.data, n, d, ctypes.byref(opts), ctypes.byref(h)))
        data.flags.writeable = False
        return cls(data, h, device=device, global_offset=int(global_offset), global_n=int(global_n or n),
                   precision=precision)

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def d(self) -> int:
        return self.data.shape[1]

    @property
    def handle(self):
        return self._handle

    @property
    def exact_mode(self) -> bool:
        """True when rows are small integers and the single-pass fp16 tile is bit-exact."""
        ex = ctypes.c_int32()
        _lib.check(_lib.load().dk_info(self._handle, None, None, None, None, ctypes.byref(ex)))
        return bool(ex.value)

    @property
    def sq_norms(self) -> np.ndarray:
        """fp64 squared row norms, computed on the device at fit (data.py:63-64)."""
        if self._sq_norms is None:
            out = np.empty(self.n, dtype=np.float64)
            _lib.check(_lib.load().dk_sq_norms(self._handle, out.ctypes.data, None))
            out.flags.writeable = False
            self._sq_norms = out
        return self._sq_norms

    def free(self) -> None:
        self._finalizer()


def _free_handle(h):
    try:
        _lib.load().dk_free(h)
    except Exception:  # interpreter shutdown
        pass


_CACHE: "weakref.WeakKeyDictionary[object, Dataset]" = weakref.WeakKeyDictionary()


def as_gpu_dataset(dataset) -> Dataset:
    """This package's Dataset, or a cached device fit of a duck-typed one."""
    if isinstance(dataset, Dataset):
        return dataset
    try:
        cached = _CACHE.get(dataset)
    except TypeError:
        cached = None
    if cached is not None:
        return cached
    data = getattr(dataset, "data", None)
    if data is None:
        raise TypeError(f"expected a Dataset-like object with a .data array, got {type(dataset)!r}")
    gpu = Dataset.from_array(data)
    try:
        _CACHE[dataset] = gpu
    except TypeError:
        pass
    return gpu


class PermutedDataset:
    """Rows reordered by a stored permutation (data.py:103-117), fitted on the device.

    ``base`` holds row ``permutation[i]`` of the original at position i, so the
    permuted sampler's windows are contiguous row ranges on the GPU; the inverse
    permutation (original id -> position) is attached to the base handle for
    excluding neighbour ids (dk_rsp_attach).
    """

    def __init__(self, base: Dataset, permutation: np.ndarray, inverse_permutation: np.ndarray):
        self.base = base
        self.permutation = permutation
        self.inverse_permutation = inverse_permutation
        inv = np.ascontiguousarray(inverse_permutation, dtype=np.int64)
        _lib.check(_lib.load().dk_rsp_attach(base.handle, inv.ctypes.data))

    @property
    def n(self) -> int:
        return self.base.n


def permute(dataset, seed: int) -> PermutedDataset:
    """Seeded Fisher-Yates reordering with numpy's PCG64, exactly as data.py:214-233."""
    ds = as_gpu_dataset(dataset)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(ds.n).astype(np.int64)
    inverse = np.empty_like(perm)
    inverse[perm] = np.arange(ds.n, dtype=np.int64)
    perm.flags.writeable = False
    inverse.flags.writeable = False
    base = Dataset.from_array(ds.data[perm], device=ds.device, precision=ds.precision)
    return PermutedDataset(base, perm, inverse)


_PCACHE: "weakref.WeakKeyDictionary[object, PermutedDataset]" = weakref.WeakKeyDictionary()


def as_gpu_permuted(permuted) -> PermutedDataset:
    """This package's PermutedDataset, or a cached device fit of the reference's one."""
    if isinstance(permuted, PermutedDataset):
        return permuted
    cached = _PCACHE.get(permuted)
    if cached is not None:
        return cached
    base = Dataset.from_array(np.asarray(permuted.base.data))
    out = PermutedDataset(base, np.asarray(permuted.permutation, dtype=np.int64),
                          np.asarray(permuted.inverse_permutation, dtype=np.int64))
    _PCACHE[permuted] = out
    return out
