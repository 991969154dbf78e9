"""batch_sqdist / window_sqdist / sqdist on the GPU (reference distance.py:42-123).

Restates the reference's own distance tests (test_distance.py) against the GPU
implementation, and compares full matrices with the oracle's restatement of the
reference's fp64 norms identity (oracle/deann_oracle.py:batch_sqdist).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

import paper_2107_02736_b200 as g
from oracle import deann_oracle as O

pytestmark = pytest.mark.gpu


def test_sqdist_scalar():
    assert g.sqdist([0.0, 0.0], [3.0, 4.0]) == 25.0
    x = np.array([1.5, -2.25, 7.0])
    assert g.sqdist(x, x) == 0.0
    with pytest.raises(ValueError):
        g.sqdist([1.0], [1.0, 2.0])
    rng = np.random.default_rng(3)
    a, b = rng.normal(size=9), rng.normal(size=9)
    exact = sum((Fraction(float(u)) - Fraction(float(v))) ** 2 for u, v in zip(a, b))
    assert g.sqdist(a, b) == pytest.approx(float(exact), rel=1e-10)


def test_batch_single_row_self_is_zero():
    row = np.array([[2.5, -1.0, 0.25]], dtype=np.float32)
    out = g.batch_sqdist(row.astype(np.float64), g.Dataset.from_array(row))
    assert out.values.shape == (1, 1) and out.values[0, 0] == 0.0
    assert out.rows == 1 and out.cols == 1


def test_batch_matches_pairwise_small_integers_exactly():
    q = np.array([[0, 0], [1, 2], [3, 3]], dtype=np.float64)
    x = np.array([[0, 0], [1, 0], [2, 2], [5, 1]], dtype=np.float32)
    out = g.batch_sqdist(q, g.Dataset.from_array(x)).values
    for j in range(3):
        for i in range(4):
            assert out[j, i] == g.sqdist(q[j], x[i])


@pytest.mark.parametrize("nq,n,d", [(20, 200, 50), (1, 1, 1), (65, 129, 17), (300, 5000, 96), (7, 3000, 784)])
def test_batch_matches_oracle_identity(nq, n, d):
    rng = np.random.default_rng(nq + n + d)
    q = rng.normal(size=(nq, d))
    x = rng.normal(size=(n, d)).astype(np.float32)
    got = g.batch_sqdist(q, g.Dataset.from_array(x)).values
    od = O.Data(x)
    ref = O.batch_sqdist(q, od.x64, od.sq_norms)
    scale = float(np.einsum("ij,ij->i", q, q).max() + od.sq_norms.max())
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(scale, 1.0))
    assert got.min() >= 0.0


def test_batch_clamps_cancellation_to_zero():
    base = np.full(32, 1e4, dtype=np.float32)
    ds = g.Dataset.from_array(np.vstack([base, base]))
    out = g.batch_sqdist(base.astype(np.float64).reshape(1, -1), ds).values
    assert out.min() >= 0.0


def test_corrupt_cached_norms_raise():
    class RefLike:  # a reference Dataset: rows plus (here corrupted) cached norms
        def __init__(self, data, sq_norms):
            self.data = data
            self.sq_norms = sq_norms

    data = np.random.default_rng(0).normal(size=(4, 3)).astype(np.float32)
    good = np.einsum("ij,ij->i", data.astype(np.float64), data.astype(np.float64))
    g.batch_sqdist(np.zeros((1, 3)), RefLike(data, good))
    with pytest.raises(g.NormConsistencyError):
        g.batch_sqdist(np.zeros((1, 3)), RefLike(data, good - 100.0))


def test_dimension_mismatch():
    ds = g.Dataset.from_array(np.ones((2, 3), dtype=np.float32))
    with pytest.raises(ValueError):
        g.batch_sqdist(np.ones((1, 4)), ds)


def test_window_sqdist_wraps_and_matches_permuted_rows():
    rng = np.random.default_rng(8)
    x = rng.normal(size=(50, 6)).astype(np.float32)
    pds = g.permute(g.Dataset.from_array(x), 3)
    y = rng.normal(size=6)
    out = g.window_sqdist(pds, 45, 10, y)
    rows = [(45 + i) % 50 for i in range(10)]
    ref = [g.sqdist(pds.base.data[r], y) for r in rows]
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        g.window_sqdist(pds, 50, 3, y)
    with pytest.raises(ValueError):
        g.window_sqdist(pds, 0, 51, y)


def test_kernel_pair_ground_truth_and_split():
    x, y = [0.0, 0.0, 0.0], [1.0, 2.0, 2.0]
    assert g.kernel_pair(g.KernelSpec("gaussian", 1.5), x, y) == pytest.approx(np.exp(-9.0 / 4.5), rel=1e-15)
    assert g.kernel_pair(g.KernelSpec("exponential", 1.5), x, y) == pytest.approx(np.exp(-2.0), rel=1e-15)
    assert g.kernel_pair(g.KernelSpec("laplacian", 2.5), x, y) == pytest.approx(np.exp(-2.0), rel=1e-15)
    with pytest.raises(ValueError):
        g.kernel_pair(g.KernelSpec("gaussian", 1.0), [1.0], [1.0, 2.0])
    X = np.random.default_rng(4).normal(size=(1200, 5)).astype(np.float32)
    sp = g.split(g.Dataset.from_array(X), 9)
    ref_order = np.random.default_rng(9).permutation(1200)   # data.py:200-206
    np.testing.assert_array_equal(sp.validation_indices, np.sort(ref_order[:500]))
    np.testing.assert_array_equal(sp.test_indices, np.sort(ref_order[500:1000]))
    assert sp.train.n == 200 and sp.validation.n == 500 and sp.test.n == 500
    np.testing.assert_array_equal(sp.train.data, X[sp.train_indices])
    gt = g.ground_truth(sp.train, X[:4].astype(np.float64), g.KernelSpec("gaussian", 1.0))
    ref = O.naive_kde(O.Data(X[sp.train_indices]), "gaussian", 1.0, X[:4].astype(np.float64))
    np.testing.assert_allclose(gt["values"], ref, rtol=1e-5)
    assert gt["n_queries"] == 4 and gt["kernel"] == "gaussian" and len(gt["dataset_sha256"]) == 64
