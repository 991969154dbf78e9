"""Edge cases across the GPU paths: odd widths (rows not whole float4s), single rows,
query-padding boundaries, underflowing and saturating bandwidths, far queries.

Every value is checked against the oracle restatement of the reference
(oracle/deann_oracle.py), with the same tolerances as the parity tests:
exact KDE 1e-5 relative (gate 1e-4), k-NN identical, RS/DEANN 1e-12 relative
given the same neighbour and sample indices.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2107_02736_b200 as g
from dk_testutil import FAMILIES
from oracle import deann_oracle as O
from oracle.philox import IndexReplay, NeighborReplay

pytestmark = pytest.mark.gpu

KDE_RTOL = 1e-5


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def _h(fam, d):
    return 2 * d ** 0.75 if fam == "laplacian" else math.sqrt(d)


@pytest.mark.parametrize("d", [1, 2, 3, 5, 7, 13, 33])
def test_odd_widths_all_paths(d):
    rng = np.random.default_rng(100 + d)
    n = 3000
    X = rng.normal(size=(n, d)).astype(np.float32)
    Q = rng.normal(size=(9, d))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    for fam in FAMILIES:
        h = _h(fam, d)
        got = g.naive_kde(ds, g.KernelSpec(fam, h), Q).values
        assert _rel(got, O.naive_kde(od, fam, h, Q)) < KDE_RTOL, (fam, d)
    k, m, seed = 20, 150, 31
    idx, d2 = g.knn_batch(ds, Q, k)
    for fam in FAMILIES:
        h = _h(fam, d)
        vals, nbr, _ = g.deann_arrays(ds, g.KernelSpec(fam, h), Q, k, m, seed=seed, export_neighbors=True)
        for j in range(len(Q)):
            ri, rd = O.brute_force_knn(od, Q[j], k)
            np.testing.assert_array_equal(nbr[j], ri)
            ref = O.deann(od, fam, h, NeighborReplay(ri, rd), Q[j], k, m, rng=IndexReplay(seed, j, n))[0]
            assert vals[j] == pytest.approx(ref, rel=1e-12), (fam, d, j)
    # permuted sampler and IVF on the same odd width
    st = g.RspState.from_dataset(ds, 3)
    ost = O.Permuted(od, 3)
    for j in range(3):
        assert g.rsp_kde(st, g.KernelSpec("gaussian", _h("gaussian", d)), Q[j], 200).value == pytest.approx(
            O.rsp_kde(ost, "gaussian", _h("gaussian", d), Q[j], 200), rel=1e-12)
    index = g.ivf_build(ds, 8, seed=d)
    cent, lists = O.ivf_build(od, 8, d)
    for j in range(3):
        ri, _ = O.ivf_query(od, cent, lists, Q[j], 10, 3)
        np.testing.assert_array_equal(g.ivf_query(index, ds, Q[j], 10, 3).indices, ri)


def test_single_row_dataset():
    X = np.array([[0.5, -1.0, 2.0]], dtype=np.float32)
    q = np.array([0.0, 0.0, 1.0])
    ds, od = g.Dataset.from_array(X), O.Data(X)
    for fam in FAMILIES:
        assert g.naive_kde(ds, g.KernelSpec(fam, 1.3), q.reshape(1, -1)).values[0] == pytest.approx(
            O.naive_kde(od, fam, 1.3, q.reshape(1, -1))[0], rel=KDE_RTOL)
    nl = g.brute_force_knn(ds, q, 1)
    assert nl.indices.tolist() == [0]
    est = g.deann(ds, g.KernelSpec("gaussian", 1.3), g.BruteForceIndex(ds), q, 1, 0)
    assert est.value == pytest.approx(O.naive_kde(od, "gaussian", 1.3, q.reshape(1, -1))[0], rel=1e-12)
    assert est.kernel_evals == 1 and not est.truncated


@pytest.mark.parametrize("nq", [1, 127, 128, 129, 255, 256, 257, 1023])
def test_query_padding_boundaries(nq):
    rng = np.random.default_rng(nq)
    X = rng.normal(size=(2000, 24)).astype(np.float32)
    Q = rng.normal(size=(nq, 24))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    got = g.naive_kde(ds, g.KernelSpec("gaussian", 4.0), Q).values
    ref = O.naive_kde(od, "gaussian", 4.0, Q)
    assert _rel(got, ref) < KDE_RTOL
    idx, _ = g.knn_batch(ds, Q, 5)
    for j in range(0, nq, max(1, nq // 7)):
        np.testing.assert_array_equal(idx[j], O.brute_force_knn(od, Q[j], 5)[0])


def test_underflow_and_saturation():
    rng = np.random.default_rng(5)
    X = rng.normal(size=(1500, 6)).astype(np.float32)
    Q = rng.normal(size=(10, 6)) + 50.0     # far from every row
    ds, od = g.Dataset.from_array(X), O.Data(X)
    for fam in FAMILIES:
        # tiny bandwidth, far queries: every kernel value underflows (exactly 0 in fp64); the
        # fp32 epilogue is exact 0 on MUFU and <= 2^-126 per polynomial term (tile_kernel.cuh),
        # both far below the parity floor of 1e-16
        got = g.naive_kde(ds, g.KernelSpec(fam, 0.05), Q).values
        ref = O.naive_kde(od, fam, 0.05, Q)
        assert np.all(ref == 0.0) and np.all(got >= 0.0) and np.all(got < 1e-37), fam
        # huge bandwidth: every kernel value ~1
        got = g.naive_kde(ds, g.KernelSpec(fam, 1e6), Q - 50.0).values
        ref = O.naive_kde(od, fam, 1e6, Q - 50.0)
        assert _rel(got, ref) < KDE_RTOL, fam


def test_large_magnitude_rows_split_encoding():
    # offsets and spreads in the thousands: the split encoding's centring/scaling
    rng = np.random.default_rng(6)
    X = (rng.normal(size=(4000, 40)) * 30 + 5000).astype(np.float32)
    Q = rng.normal(size=(16, 40)) * 30 + 5000
    ds, od = g.Dataset.from_array(X), O.Data(X)
    for fam in ("gaussian", "exponential"):
        h = 150.0 if fam == "gaussian" else 80.0
        got = g.naive_kde(ds, g.KernelSpec(fam, h), Q).values
        assert _rel(got, O.naive_kde(od, fam, h, Q)) < KDE_RTOL, fam


def test_integer_dataset_with_fractional_queries_and_duplicates():
    rng = np.random.default_rng(7)
    X = rng.integers(0, 4, size=(3000, 10)).astype(np.float32)   # exact-mode rows, many duplicates
    Q = rng.integers(0, 4, size=(12, 10)).astype(np.float64)
    Q[6:] += 0.25                                                  # fractional half: split encoding
    ds, od = g.Dataset.from_array(X), O.Data(X)
    assert ds.exact_mode
    got = g.naive_kde(ds, g.KernelSpec("gaussian", 1.5), Q).values
    assert _rel(got, O.naive_kde(od, "gaussian", 1.5, Q)) < KDE_RTOL
    idx, _ = g.knn_batch(ds, Q, 40)
    for j in range(len(Q)):
        np.testing.assert_array_equal(idx[j], O.brute_force_knn(od, Q[j], 40)[0])


def test_very_wide_rows():
    # d = 4100: the split3 tile streams its A operand, the gather kernels run fewer queries per block
    rng = np.random.default_rng(9)
    n, d = 1500, 4100
    X = rng.normal(size=(n, d)).astype(np.float32)
    Q = X[:4].astype(np.float64) + rng.normal(scale=0.5, size=(4, d))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    for fam, h in (("gaussian", 40.0), ("exponential", 30.0), ("laplacian", 2000.0)):
        got = g.naive_kde(ds, g.KernelSpec(fam, h), Q).values
        assert _rel(got, O.naive_kde(od, fam, h, Q)) < KDE_RTOL, fam
        vals, nbr, _ = g.deann_arrays(ds, g.KernelSpec(fam, h), Q, 10, 100, seed=3, export_neighbors=True)
        for j in range(len(Q)):
            ri, rd = O.brute_force_knn(od, Q[j], 10)
            np.testing.assert_array_equal(nbr[j], ri)
            ref = O.deann(od, fam, h, NeighborReplay(ri, rd), Q[j], 10, 100, rng=IndexReplay(3, j, n))[0]
            assert vals[j] == pytest.approx(ref, rel=1e-12)
    st, ost = g.RspState.from_dataset(ds, 2), O.Permuted(od, 2)
    assert g.rsp_kde(st, g.KernelSpec("gaussian", 40.0), Q[0], 300).value == pytest.approx(
        O.rsp_kde(ost, "gaussian", 40.0, Q[0], 300), rel=1e-12)


def test_pinned_result_buffers_lifecycle():
    # results >= 1 MiB come back in page-locked buffers from the library's cache; an array
    # (or a view of it) keeps its buffer alive, and freed buffers are reused
    import gc

    from paper_2107_02736_b200 import _lib

    a = _lib.host_empty((512, 300), np.float64)
    assert a.shape == (512, 300) and a.dtype == np.float64
    a[:] = 3.0
    v = a[10:20, 5]
    del a
    gc.collect()
    assert (v == 3.0).all()
    del v
    gc.collect()
    b = _lib.host_empty((300, 512), np.int64)
    b[:] = 7
    assert int(b.sum()) == 7 * 300 * 512
    assert _lib.host_empty((4, 4), np.float64).flags.owndata  # small: plain numpy
    rng = np.random.default_rng(5)
    X = rng.normal(size=(5000, 24)).astype(np.float32)
    Q = rng.normal(size=(1500, 24))
    ds = g.Dataset.from_array(X)
    idx, d2 = g.knn_batch(ds, Q, 100)          # 1.2 MB outputs: pinned path
    idx2, d22 = g.knn_batch(ds, Q[:7], 100)    # small: numpy path
    np.testing.assert_array_equal(idx[:7], idx2)
    np.testing.assert_array_equal(d2[:7], d22)


def _redo_count(ds) -> int:
    import ctypes

    from paper_2107_02736_b200 import _lib

    c = ctypes.c_int64(-1)
    _lib.check(_lib.load().dk_kde_redo_count(ds.handle, ctypes.byref(c)))
    return int(c.value)


@pytest.mark.parametrize("n,d,scale,h", [(392, 3, 1.0, 0.075), (219, 16, 1.0, 0.19), (5000, 129, 1.0, 2.4),
                                         (13000, 16, 30.0, 25.0), (70000, 1, 1.0, 0.14)])
def test_exponential_queries_on_data_points(n, d, scale, h):
    """exp(-sqrt(d2)/h) at a (near-)coincident pair amplifies the sweep's d2 error to sqrt(eps)/h: the
    guard re-evaluates those queries in fp64 direct differences (redo.cu), as naive_kde
    (estimators.py:144-149) evaluates every pair.  Unguarded, these cases are off by 2e-4 .. 5e-3."""
    rng = np.random.default_rng(n + d)
    X = (rng.normal(size=(n, d)) * scale).astype(np.float32)
    if d == 3:
        X = np.where(rng.random((n, d)) < 0.8, 0.0, rng.random((n, d))).astype(np.float32)
    Q = X[rng.integers(0, n, size=200)].astype(np.float64)
    ds = g.Dataset.from_array(X)
    got = g.naive_kde(ds, g.KernelSpec("exponential", h), Q).values
    assert _redo_count(ds) == 200
    ref = O.naive_kde(O.Data(X), "exponential", h, Q)
    assert _rel(got, ref) < 5e-6  # the reference's own d2 (norms identity) is good to ~1e-15 |x|^2 at a coincident pair
    if d == 1:
        return  # 70,000 points on a line: every query has a row within any threshold
    # queries away from the rows stay on the tensor-core sweep
    far = Q + 3.0 * scale
    got = g.naive_kde(ds, g.KernelSpec("exponential", 40.0 * h), far).values
    assert _redo_count(ds) == 0
    assert _rel(got, O.naive_kde(O.Data(X), "exponential", 40.0 * h, far)) < KDE_RTOL


def test_gaussian_bandwidth_narrow_against_the_norms():
    """2h^2 = 4 on sparse 784-dimensional rows (|x|^2 ~ 50, K = 2352): the fp32 accumulation error of
    d2, ~5e-4, is 1.2e-4 of 2h^2, so the whole batch takes the fp64 path (1.1e-4 unguarded)."""
    rng = np.random.default_rng(359)
    n, d = 6000, 784
    X = np.where(rng.random((n, d)) < 0.8, 0.0, rng.random((n, d))).astype(np.float32)
    Q = np.where(rng.random((64, d)) < 0.8, 0.0, rng.random((64, d)))
    ds = g.Dataset.from_array(X)
    got = g.naive_kde(ds, g.KernelSpec("gaussian", 1.42), Q).values
    assert _redo_count(ds) == 64
    assert _rel(got, O.naive_kde(O.Data(X), "gaussian", 1.42, Q)) < 1e-9
    # a bandwidth in proportion to the data stays on the sweep
    got = g.naive_kde(ds, g.KernelSpec("gaussian", 6.0), Q).values
    assert _redo_count(ds) == 0
    assert _rel(got, O.naive_kde(O.Data(X), "gaussian", 6.0, Q)) < KDE_RTOL


def test_guard_on_dataset_shards():
    """A shard handle's recomputed queries carry the shard's sum scaled by the global row count."""
    rng = np.random.default_rng(5)
    n, d, h = 3000, 8, 0.3
    X = rng.normal(size=(n, d)).astype(np.float32)
    Q = X[:50].astype(np.float64)
    parts = [g.Dataset.from_array(X[lo:hi], global_offset=lo, global_n=n) for lo, hi in [(0, 1200), (1200, n)]]
    total = sum(g.naive_kde(p, g.KernelSpec("exponential", h), Q).values for p in parts)
    assert _redo_count(parts[0]) == 50
    assert _rel(total, O.naive_kde(O.Data(X), "exponential", h, Q)) < 1e-6  # the unflagged shard is a sweep


def test_knn_overflow_fallback_in_row_slices(monkeypatch):
    """20,000 copies of one row overflow a query's candidate list (cap 8,192): the query takes the exact
    fp64 scan, cut into row slices over the whole GPU on datasets of >= 131,072 rows and merged by
    (d2, index) — ties to the lower index as _smallest_k (ann.py:82-102)."""
    import ctypes

    from paper_2107_02736_b200 import _lib

    rng = np.random.default_rng(11)
    n, d, k = 140_000, 8, 10
    X = rng.normal(size=(n, d)).astype(np.float32)
    dup = rng.choice(n, size=20_000, replace=False)
    X[dup] = X[dup[0]]
    Q = np.vstack([X[dup[0]].astype(np.float64) + 1e-3, rng.normal(size=(40, d))])
    monkeypatch.setenv("DK_KNN_STATS", "1")  # read at fit time: the handle counts its fallbacks
    ds = g.Dataset.from_array(X)
    od = O.Data(X)
    idx, d2 = g.knn_batch(ds, Q, k)
    v = [ctypes.c_int64(0) for _ in range(4)]
    _lib.check(_lib.load().dk_knn_stats(ds.handle, *[ctypes.byref(x) for x in v]))
    assert v[3].value >= 1  # the duplicated-row query overflowed
    for j in range(Q.shape[0]):
        ri, rd = O.brute_force_knn(od, Q[j], k)
        if j > 0:
            np.testing.assert_array_equal(idx[j], ri)
        np.testing.assert_allclose(d2[j], rd, rtol=1e-9, atol=1e-12)
    # the 20,000 copies are exactly tied: the lower indices win here; the reference's order among them
    # follows the rounding of its BLAS matvec (the north star's "identical up to ties within 1e-6")
    np.testing.assert_array_equal(idx[0], np.sort(dup)[:k])


@pytest.mark.parametrize("family,h", [("gaussian", 1.2), ("exponential", 0.12), ("laplacian", 0.2)])
def test_far_queries_below_the_fp32_range(family, h):
    """KDE values under ~1e-38 cannot come out of the fp32 epilogue (flushed exponentials; the polynomial's
    clamp leaves ~1.5e-39): such queries are recomputed in fp64 and match the reference's tiny values."""
    rng = np.random.default_rng(77)
    X = rng.normal(size=(3000, 3)).astype(np.float32)
    Q = np.vstack([rng.normal(size=(20, 3)), rng.normal(size=(20, 3)) + 14.0])  # 20 ordinary, 20 far away
    ds = g.Dataset.from_array(X)
    got = g.naive_kde(ds, g.KernelSpec(family, h), Q).values
    ref = O.naive_kde(O.Data(X), family, h, Q)
    assert ref[20:].max() < 1e-40 and ref[20:].min() > 1e-290
    assert _redo_count(ds) >= 20
    assert _rel(got[20:], ref[20:]) < 1e-9
    ordinary = ref[:20] > 1e-30
    assert _rel(got[:20][ordinary], ref[:20][ordinary]) < KDE_RTOL
