"""CPU: the C-ABI library loads, exports every declared symbol, and rejects bad
arguments with the reference's ValueError preconditions before touching a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2107_02736_b200 import _lib
from dk_testutil import REPO

HEADER = os.path.join(REPO, "include", "deann_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dk_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    lib = _lib.load()
    assert lib.dk_version() >= 10000


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == declared


def test_null_handle_is_einval():
    lib = _lib.load()
    out = np.zeros(1)
    q = np.zeros((1, 2))
    st = lib.dk_naive(None, q.ctypes.data, 1, 0, 1.0, 0, out.ctypes.data, None)
    assert st == _lib.DK_EINVAL
    assert "NULL" in lib.dk_last_error().decode()


@pytest.mark.parametrize("bw", [0.0, -1.0, float("inf"), float("nan")])
def test_bad_bandwidth_is_valueerror(bw):
    lib = _lib.load()
    d = np.ones(3)
    out = np.empty(3)
    with pytest.raises(ValueError, match="bandwidth"):
        _lib.check(lib.dk_kernel_values(0, bw, d.ctypes.data, 3, out.ctypes.data, None))


def test_bad_family_is_valueerror():
    lib = _lib.load()
    d = np.ones(3)
    out = np.empty(3)
    with pytest.raises(ValueError, match="family"):
        _lib.check(lib.dk_kernel_values(7, 1.0, d.ctypes.data, 3, out.ctypes.data, None))


def test_fit_shape_errors():
    lib = _lib.load()
    h = ctypes.c_void_p()
    x = np.zeros((1, 1), dtype=np.float32)
    with pytest.raises(ValueError, match="n >= 1 and d >= 1"):
        _lib.check(lib.dk_fit(x.ctypes.data, 0, 4, None, ctypes.byref(h)))
    with pytest.raises(ValueError, match="n >= 1 and d >= 1"):
        _lib.check(lib.dk_fit(x.ctypes.data, 4, 0, None, ctypes.byref(h)))


def test_merge_argument_errors():
    lib = _lib.load()
    with pytest.raises(ValueError):
        _lib.check(lib.dk_merge_topk(0, 1, 1, None, None, None, None, None))


def test_python_dataset_validation_before_gpu():
    from paper_2107_02736_b200 import Dataset

    with pytest.raises(ValueError, match="2-dimensional"):
        Dataset.from_array(np.zeros(5, dtype=np.float32))
    with pytest.raises(ValueError, match="n >= 1"):
        Dataset.from_array(np.zeros((0, 3), dtype=np.float32))
    with pytest.raises(ValueError, match="precision"):
        Dataset.from_array(np.zeros((2, 3), dtype=np.float32), precision="bogus")


def test_kernel_spec_validation():
    from paper_2107_02736_b200 import KernelFamily, KernelSpec

    assert KernelSpec("gaussian", 2).bandwidth == 2.0
    assert KernelSpec("laplacian", 1.0).metric == "l1"
    assert KernelFamily("exponential").metric == "l2"
    for bad in (0.0, -2.0, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            KernelSpec("gaussian", bad)
    with pytest.raises(ValueError):
        KernelSpec("cauchy", 1.0)


def test_deann_preconditions_match_reference():
    # estimators.py:322-335 (checked on the host before any launch)
    from paper_2107_02736_b200.estimators import _validate

    rng = np.random.default_rng(0)

    class _Rsp:
        n = 19

    with pytest.raises(ValueError):
        _validate(20, 2, 21, 0, None, None)
    with pytest.raises(ValueError):
        _validate(20, 2, 20, 5, rng, None)
    with pytest.raises(ValueError):
        _validate(20, 2, 2, -1, rng, None)
    with pytest.raises(ValueError):
        _validate(20, 2, 2, 5, None, None)
    with pytest.raises(ValueError):
        _validate(20, 2, 2, 5, rng, _Rsp())
    with pytest.raises(ValueError):
        _validate(20, 2, 2, 5, None, _Rsp())
    _validate(20, 2, 0, 5, rng, None)
    _validate(20, 2, 20, 0, None, None)


def test_sampler_resolution():
    from paper_2107_02736_b200 import PhiloxSampler
    from paper_2107_02736_b200.sampler import resolve_sampler

    a = resolve_sampler(np.random.default_rng(77))
    b = resolve_sampler(np.random.default_rng(77))
    assert a.seed == b.seed
    s = PhiloxSampler(5)
    assert s.take(3) == (5, 0) and s.take(2) == (5, 3)
    assert resolve_sampler(s) is s
    with pytest.raises(TypeError):
        resolve_sampler("nope")
