"""ctypes binding of the C-ABI library ``libdeann_b200.so`` (include/deann_b200.h).

The product path has no CPU fallback: if the library is missing or no sm_100
device is present, every estimator raises.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make`` in
``paper_2107_02736_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DK_LIBRARY") or os.path.join(_HERE, "libdeann_b200.so")

DK_OK, DK_EINVAL, DK_ECUDA, DK_ENOMEM, DK_EINEXACT, DK_ENODEV, DK_EFORMAT, DK_EIO = range(8)
DK_GAUSSIAN, DK_EXPONENTIAL, DK_LAPLACIAN = 0, 1, 2
DK_PREC_AUTO, DK_PREC_SPLIT3, DK_PREC_FP16 = 0, 1, 2
DK_OUT_SUM = 1

# every symbol include/deann_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "dk_version", "dk_last_error", "dk_device_ok", "dk_fit", "dk_free", "dk_file_info", "dk_fit_file",
    "dk_info", "dk_sq_norms",
    "dk_naive", "dk_sqdist", "dk_knn", "dk_merge_topk", "dk_sample", "dk_eval_rows", "dk_kernel_values", "dk_deann",
    "dk_rsp_attach", "dk_rsp_walk", "dk_ivf_create", "dk_ivf_free", "dk_kmeanspp_seed", "dk_kmeanspp_pick",
    "dk_kmeans_lloyd", "dk_ivf_get", "dk_ivf_set", "dk_ivf_query", "dk_last_kernel_ms", "dk_set_profiling", "dk_last_launch_count", "dk_knn_stats", "dk_kde_stats", "dk_kde_redo_count", "dk_sweep_probe",
    "dk_host_alloc", "dk_host_free", "dk_deann_ivf", "dk_deann_combine", "dk_mufu_probe",
)


class DeannGpuError(RuntimeError):
    """A CUDA / device failure reported by the C-ABI (status DK_ECUDA / DK_ENODEV)."""


class DatasetFormatError(ValueError):
    """A dataset file cannot be parsed (reference data.DatasetFormatError, data.py:41-42)."""


class FitOpts(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("global_offset", ctypes.c_int64),
        ("global_n", ctypes.c_int64),
    ]


_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_f64 = ctypes.c_double


def _declare(lib):
    sig = {
        "dk_version": (_i32, []),
        "dk_last_error": (ctypes.c_char_p, []),
        "dk_device_ok": (_i32, [_i32]),
        "dk_fit": (_i32, [_vp, _i64, _i32, ctypes.POINTER(FitOpts), ctypes.POINTER(_vp)]),
        "dk_free": (_i32, [_vp]),
        "dk_sqdist": (_i32, [_vp, _vp, _i64, _vp, _i64, _i64, _vp, ctypes.POINTER(_f64), _vp]),
        "dk_ivf_create": (_i32, [_vp, _i32, ctypes.POINTER(_vp)]),
        "dk_ivf_free": (_i32, [_vp]),
        "dk_kmeanspp_seed": (_i32, [_vp, _i32, _i64, ctypes.POINTER(_f64)]),
        "dk_kmeanspp_pick": (_i32, [_vp, _f64, _f64, ctypes.POINTER(_i64)]),
        "dk_kmeans_lloyd": (_i32, [_vp, _i32, _f64, ctypes.POINTER(_i32)]),
        "dk_ivf_get": (_i32, [_vp, _vp, _vp, _vp]),
        "dk_ivf_set": (_i32, [_vp, _vp, _vp, _vp]),
        "dk_ivf_query": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
        "dk_deann_ivf": (_i32, [_vp, _vp, _i64, _i32, _f64, _i32, _i32, _i32, _u64, _i64, _vp, _vp, _vp]),
        "dk_file_info": (_i32, [ctypes.c_char_p, ctypes.POINTER(_i64), ctypes.POINTER(_i32)]),
        "dk_fit_file": (_i32, [ctypes.c_char_p, _i64, _i64, ctypes.POINTER(FitOpts), ctypes.POINTER(_vp)]),
        "dk_info": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i64),
                            ctypes.POINTER(_i64), ctypes.POINTER(_i32)]),
        "dk_sq_norms": (_i32, [_vp, _vp, _vp]),
        "dk_naive": (_i32, [_vp, _vp, _i64, _i32, _f64, _u32, _vp, _vp]),
        "dk_knn": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp]),
        "dk_merge_topk": (_i32, [_i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
        "dk_sample": (_i32, [_vp, _vp, _i64, _i32, _f64, _i32, _u64, _i64, _vp, _vp, _i32, _vp, _vp, _vp, _vp]),
        "dk_eval_rows": (_i32, [_vp, _vp, _i64, _i32, _f64, _vp, _vp, _i32, _vp, _vp]),
        "dk_kernel_values": (_i32, [_i32, _f64, _vp, _i64, _vp, _vp]),
        "dk_deann": (_i32, [_vp, _vp, _i64, _i32, _f64, _i32, _i32, _u64, _i64, _vp, _vp, _vp, _vp, _vp]),
        "dk_mufu_probe": (_i32, [_i32, ctypes.POINTER(_f64)]),
        "dk_deann_combine": (_i32, [_i64, _i32, _f64, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp]),
        "dk_rsp_attach": (_i32, [_vp, _vp]),
        "dk_rsp_walk": (_i32, [_vp, _vp, _i64, _i32, _f64, _i32, _vp, _i32, _i64, _i32, _vp, _vp,
                                ctypes.POINTER(_i64), _vp]),
        "dk_last_kernel_ms": (_i32, [_vp, ctypes.POINTER(_f64), ctypes.POINTER(_f64), ctypes.POINTER(_f64)]),
        "dk_set_profiling": (_i32, [_vp, _i32]),
        "dk_last_launch_count": (_i32, [_vp, ctypes.POINTER(_i64)]),
        "dk_sweep_probe": (_i32, [_vp, _vp, _i64, _i32, _i32, ctypes.POINTER(_f64)]),
        "dk_knn_stats": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                ctypes.POINTER(_i64)]),
        "dk_kde_stats": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                ctypes.POINTER(_i64)]),
        "dk_kde_redo_count": (_i32, [_vp, ctypes.POINTER(_i64)]),
        "dk_host_alloc": (_i32, [_i64, ctypes.POINTER(_vp)]),
        "dk_host_free": (_i32, [_vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load():
    """Load the C-ABI library (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} not found: the CUDA extension is not built "
                    "(run `make -C paper_2107_02736_b200/csrc` or __graft_entry__.build())"
                )
            _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def check(status: int) -> None:
    if status == DK_OK:
        return
    msg = load().dk_last_error().decode(errors="replace")
    if status == DK_EINVAL:
        raise ValueError(msg)
    if status == DK_EFORMAT:
        raise DatasetFormatError(msg)
    if status == DK_EIO:
        raise OSError(msg)
    if status == DK_ENOMEM:
        raise MemoryError(msg)
    raise DeannGpuError(f"[status {status}] {msg}")


def ptr(obj) -> int | None:
    """Raw address of a numpy array or torch tensor (None passes through)."""
    if obj is None:
        return None
    if isinstance(obj, np.ndarray):
        return obj.ctypes.data
    if hasattr(obj, "data_ptr"):
        return obj.data_ptr()
    raise TypeError(f"cannot take the address of {type(obj)!r}")


def current_stream():
    """cudaStream_t of torch's current stream when torch is loaded, else the default stream."""
    import sys

    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        return torch.cuda.current_stream().cuda_stream
    return None


class _PinnedBlock:
    """One dk_host_alloc buffer, returned to the library's cache when collected."""

    __slots__ = ("ptr",)

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        check(load().dk_host_alloc(nbytes, ctypes.byref(p)))
        self.ptr = p.value

    def __del__(self):
        try:
            load().dk_host_free(ctypes.c_void_p(self.ptr))
        except Exception:  # interpreter shutdown
            pass


def host_empty(shape, dtype) -> np.ndarray:
    """Uninitialised host output array; large ones (1 MiB .. 512 MiB) live in page-locked memory
    from the library's cache (dk_host_alloc), so device->host copies of results run at
    full DMA speed instead of through a pageable bounce buffer.  The array (and any view
    of it) keeps the buffer alive."""
    dt = np.dtype(dtype)
    shape = tuple(int(x) for x in np.atleast_1d(shape))
    count = int(np.prod(shape, dtype=np.int64))
    nbytes = count * dt.itemsize
    if nbytes < (1 << 20) or nbytes > (1 << 29):  # small, or too big to pin by power-of-two classes
        return np.empty(shape, dtype=dt)
    try:
        block = _PinnedBlock(nbytes)
    except (MemoryError, DeannGpuError):
        return np.empty(shape, dtype=dt)
    buf = (ctypes.c_char * nbytes).from_address(block.ptr)
    buf._dk_block = block
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


def family_code(family) -> int:
    v = getattr(family, "value", family)
    return {"gaussian": DK_GAUSSIAN, "exponential": DK_EXPONENTIAL, "laplacian": DK_LAPLACIAN}[str(v)]
