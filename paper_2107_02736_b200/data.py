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
import os
import struct
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["Dataset", "as_gpu_dataset", "PermutedDataset", "permute", "as_gpu_permuted", "DatasetFormatError",
           "file_info", "load", "save", "Splits", "split"]

DatasetFormatError = _lib.DatasetFormatError
MAGIC = b"DEANN1\x00\x00"
HEADER_BYTES = 16

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
        self._data64 = None
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

    def data64(self) -> np.ndarray:
        """Read-only fp64 copy of the host rows, cached after first use (data.py:77-83).

        Not used by any estimator here (the device holds the rows); provided for the
        reference's own callers (harness.py:247, analysis.py:215-283, cli.py:148-200)."""
        if self._data64 is None:
            d64 = np.asarray(self.data).astype(np.float64)
            d64.flags.writeable = False
            self._data64 = d64
        return self._data64

    def free(self) -> None:
        self._finalizer()

    def take(self, indices) -> "Dataset":
        """New fitted dataset from a row subset (data.py:85-87; norms recomputed on the device)."""
        return Dataset.from_array(self.data[np.asarray(indices, dtype=np.intp)], device=self.device,
                                  precision=self.precision)


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


# ---------------------------------------------------------------- files


def file_info(path) -> tuple[int, int]:
    """(n, d) of a DEANN1 file; header and payload size validated as data.py:151-167."""
    with open(path, "rb"):  # FileNotFoundError / PermissionError exactly as the reference's open()
        pass
    n, d = ctypes.c_int64(), ctypes.c_int32()
    _lib.check(_lib.load().dk_file_info(os.fsencode(path), ctypes.byref(n), ctypes.byref(d)))
    return int(n.value), int(d.value)


def load(path, fmt: str = "binary", *, device: int = 0, precision: str = "auto", rows=None) -> Dataset:
    """Read a dataset file (reference data.load, data.py:142-148) straight onto the GPU.

    binary: the header is validated by the C-ABI (same DatasetFormatError messages
    as the reference), the rows stream from the file through pinned buffers into
    device memory (dk_fit_file), and ``.data`` is a read-only memory map of the
    file — no host copy is made.  ``rows=(begin, count)`` loads a row range as a
    dataset shard whose global ids are the file's row ids.
    csv: parsed on the host exactly like data.py:170-190, then uploaded.
    """
    if fmt == "binary":
        return _load_binary(path, device, precision, rows)
    if fmt == "csv":
        if rows is not None:
            raise ValueError("rows= is only supported for binary files")
        return Dataset.from_array(_parse_csv(path), device=device, precision=precision)
    raise ValueError(f"unknown format {fmt!r}")


def _load_binary(path, device, precision, rows) -> Dataset:
    if precision not in _PRECISION:
        raise ValueError(f"precision must be one of {sorted(_PRECISION)}, got {precision!r}")
    n, d = file_info(path)
    begin, count = (0, n) if rows is None else (int(rows[0]), int(rows[1]))
    if not (0 <= begin and 1 <= count and begin + count <= n):
        raise ValueError(f"row range [{begin}, {begin + count}) outside the file's {n} rows")
    data = np.memmap(path, dtype="<f4", mode="r", offset=HEADER_BYTES + begin * d * 4, shape=(count, d))
    shard = count < n
    opts = _lib.FitOpts(device, _PRECISION[precision], begin if shard else 0, n if shard else 0)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().dk_fit_file(os.fsencode(path), begin, count, ctypes.byref(opts), ctypes.byref(h)))
    return Dataset(data, h, device=device, global_offset=begin if shard else 0, global_n=n, precision=precision)


def _parse_csv(path) -> np.ndarray:
    rows = []
    width = None
    with open(path, "r") as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if width is None:
                width = len(parts)
            elif len(parts) != width:
                raise DatasetFormatError(f"{path}: line {lineno} has {len(parts)} fields, expected {width}")
            try:
                rows.append([float(p) for p in parts])
            except ValueError as exc:
                raise DatasetFormatError(f"{path}: line {lineno}: {exc}") from exc
    if not rows:
        raise DatasetFormatError(f"{path}: no data rows")
    return np.asarray(rows, dtype=np.float32)


def save(dataset, path, fmt: str = "binary") -> None:
    """Write a dataset (reference data.save, data.py:131-139); binary is bit-exact."""
    data = np.asarray(getattr(dataset, "data", dataset))
    if fmt == "binary":
        with open(path, "wb") as f:
            f.write(MAGIC + struct.pack("<II", data.shape[0], data.shape[1]))
            f.write(np.ascontiguousarray(data, dtype="<f4").tobytes())
    elif fmt == "csv":
        np.savetxt(path, data, delimiter=",", fmt="%.9g")
    else:
        raise ValueError(f"unknown format {fmt!r}")


# ---------------------------------------------------------------- splits (data.py:90-101, 192-211)


@dataclass
class Splits:
    """Disjoint train/validation/test parts whose union is the input."""

    train: Dataset
    validation: Dataset
    test: Dataset
    seed: int
    train_indices: np.ndarray
    validation_indices: np.ndarray
    test_indices: np.ndarray


def split(dataset, seed: int) -> Splits:
    """Seeded disjoint split with numpy's PCG64, identical to the reference's (data.py:192-211):
    up to 500 validation and 500 test rows, the rest training (at least one row)."""
    ds = as_gpu_dataset(dataset)
    n = ds.n
    if n <= 2:
        raise ValueError(f"cannot split a dataset with n={n}; need n > 2")
    n_val = min(500, n - 2)
    n_test = min(500, n - n_val - 1)
    order = np.random.default_rng(seed).permutation(n)
    val_idx = np.sort(order[:n_val])
    test_idx = np.sort(order[n_val:n_val + n_test])
    train_idx = np.sort(order[n_val + n_test:])
    return Splits(train=ds.take(train_idx), validation=ds.take(val_idx), test=ds.take(test_idx), seed=seed,
                  train_indices=train_idx, validation_indices=val_idx, test_indices=test_idx)
