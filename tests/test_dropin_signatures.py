"""CPU: the drop-in mirrors the REAL reference's public hot-path surface.

Imports the reference package read-only from /root/reference/pkg/src (present in
the build container, absent on the GPU box -> skipped there) and checks, symbol
by symbol, that every reference parameter exists in the drop-in with the same
name, kind, position and default (the drop-in may only ADD keyword-only
parameters with defaults), and that the attributes the reference's own callers
read exist (harness.py:243-256, analysis.py:215-283, cli.py:148-200).
"""

import importlib
import inspect
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "deann")),
                                reason="reference checkout not present (GPU box)")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF_SRC)
    try:
        return importlib.import_module("deann")
    finally:
        sys.path.remove(REF_SRC)


@pytest.fixture(scope="module")
def ours():
    return importlib.import_module("paper_2107_02736_b200")


# the hot-path public symbols of the reference (deann/__init__.py:8-43) the drop-in serves
FUNCS = [
    "naive_kde", "rs_kde", "rsp_kde", "deann", "deann_batch", "brute_force_knn", "kernel_from_distance",
    "kernel_pair", "batch_sqdist", "sqdist", "window_sqdist", "fit_bandwidth", "ivf_build", "ivf_query",
    "recall", "save_ivf_index", "load_ivf_index", "load", "save", "permute", "split", "ground_truth",
]
METHODS = [
    ("Dataset", "from_array"), ("Dataset", "data64"), ("Dataset", "take"),
    ("RspState", "from_dataset"), ("AnnIndex", "query"), ("BruteForceIndex", "query"),
    ("BruteForceIndex", "__init__"), ("IvfAnnIndex", "__init__"), ("IvfAnnIndex", "query"),
    ("IvfAnnIndex", "build"), ("NeighborList", "__init__"), ("Estimate", "__init__"), ("BatchKde", "__init__"),
    ("KernelSpec", "__init__"),
]


def _compatible(rsig: inspect.Signature, osig: inspect.Signature, what: str):
    rp = list(rsig.parameters.values())
    op = list(osig.parameters.values())
    assert len(op) >= len(rp), f"{what}: drop-in drops parameters {rsig} vs {osig}"
    for a, b in zip(rp, op):
        assert a.name == b.name, f"{what}: parameter {a.name!r} is named {b.name!r} in the drop-in"
        assert a.kind == b.kind, f"{what}: parameter {a.name!r} kind {a.kind} vs {b.kind}"
        assert a.default == b.default or (a.default is inspect.Parameter.empty) == (b.default is inspect.Parameter.empty) \
            and a.default == b.default, f"{what}: default of {a.name!r} is {a.default!r} vs {b.default!r}"
    for b in op[len(rp):]:
        assert b.kind in (inspect.Parameter.KEYWORD_ONLY, inspect.Parameter.VAR_KEYWORD) or \
            b.default is not inspect.Parameter.empty, f"{what}: extra parameter {b.name!r} must be optional"


@pytest.mark.parametrize("name", FUNCS)
def test_function_signature(ref, ours, name):
    assert hasattr(ours, name), f"drop-in is missing {name}"
    _compatible(inspect.signature(getattr(ref, name)), inspect.signature(getattr(ours, name)), name)


@pytest.mark.parametrize("cls,meth", METHODS)
def test_method_signature(ref, ours, cls, meth):
    rc, oc = getattr(ref, cls), getattr(ours, cls)
    assert hasattr(oc, meth), f"drop-in {cls} is missing {meth}"
    _compatible(inspect.signature(getattr(rc, meth)), inspect.signature(getattr(oc, meth)), f"{cls}.{meth}")


def test_kernel_family_members(ref, ours):
    assert {m.name: m.value for m in ref.KernelFamily} == {m.name: m.value for m in ours.KernelFamily}
    for m in ref.KernelFamily:
        assert ours.KernelFamily[m.name].metric == m.metric


def test_result_record_fields(ref, ours):
    import dataclasses

    for cls in ("Estimate", "BatchKde", "NeighborList"):
        rf = [(f.name, f.default) for f in dataclasses.fields(getattr(ref, cls))]
        of = [(f.name, f.default) for f in dataclasses.fields(getattr(ours, cls))]
        assert rf == of, cls


def test_attributes_the_reference_callers_read(ref, ours):
    """harness._Runner.warm reads train.data64() and ann._vectors32 (harness.py:247-249);
    analysis.fit_bandwidth reads data64() (analysis.py:283); cli reads .n/.d/.data."""
    import numpy as np

    X = (np.arange(48, dtype=np.float32).reshape(12, 4) % 7)
    ds = ours.Dataset.__new__(ours.Dataset)  # no device: attributes only
    ds.data = X
    ds._data64 = None
    d64 = ours.Dataset.data64(ds)
    assert d64.dtype == np.float64 and np.array_equal(d64, X.astype(np.float64)) and not d64.flags.writeable
    assert ours.Dataset.data64(ds) is d64  # cached like data.py:77-83
    for attr in ("data", "sq_norms", "n", "d", "data64", "take"):
        assert hasattr(ours.Dataset, attr) or attr == "data"
    for attr in ("dataset", "index", "n_probe", "_vectors32", "_row_ids", "_norms32", "_offsets"):
        assert attr in ours.IvfAnnIndex.__init__.__code__.co_names or hasattr(ours.IvfAnnIndex, attr), attr
    for attr in ("permuted", "cursor", "n"):
        assert hasattr(ours.RspState, attr) or attr in [f.name for f in __import__("dataclasses").fields(ours.RspState)]
