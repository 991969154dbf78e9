"""Large k (> 4096) and long exclusion lists (> 16384 ids) on the GPU.

The reference accepts any 1 <= k <= n (ann.py:107-108) and excludes the whole
neighbour set from the sampler (estimators.py:215-233), so these sizes must
give the same answers as the small-k tile path: exact neighbours with the
lower-index tie break and bit-identical sampler streams.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2107_02736_b200 as g
from oracle import deann_oracle as O
from oracle.philox import IndexReplay, NeighborReplay

pytestmark = pytest.mark.gpu


def _tied_rows(n, d, seed):
    rng = np.random.default_rng(seed)
    X = rng.integers(-3, 4, size=(n, d)).astype(np.float32)  # many exactly equal distances
    X[n // 2:] += rng.normal(scale=0.25, size=(n - n // 2, d)).astype(np.float32)
    return X


@pytest.mark.parametrize("k", [4097, 6500, 9000])
def test_knn_large_k_matches_oracle_with_ties(k):
    X = _tied_rows(9000, 6, 3)
    Q = np.random.default_rng(4).normal(size=(3, 6))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    idx, d2 = g.knn_batch(ds, Q, k)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], k)
        np.testing.assert_array_equal(idx[j], ri)
        np.testing.assert_allclose(d2[j], rd, rtol=1e-12, atol=0)


def test_knn_boundary_k_4096_and_4097_agree():
    X = np.random.default_rng(5).normal(size=(12_000, 20)).astype(np.float32)
    Q = np.random.default_rng(6).normal(size=(4, 20))
    ds = g.Dataset.from_array(X)
    i1, d1 = g.knn_batch(ds, Q, 4096)
    i2, d2 = g.knn_batch(ds, Q, 4097)
    np.testing.assert_array_equal(i1, i2[:, :4096])
    np.testing.assert_allclose(d1, d2[:, :4096], rtol=1e-12)


def test_knn_k_3000_mid_size_n():
    # too few segment minima to bound tau for this k: the plan falls back to the exact path
    X = np.random.default_rng(16).normal(size=(100_000, 12)).astype(np.float32)
    Q = np.random.default_rng(17).normal(size=(2, 12))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    idx, d2 = g.knn_batch(ds, Q, 3000)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], 3000)
        np.testing.assert_array_equal(idx[j], ri)
        np.testing.assert_allclose(d2[j], rd, rtol=1e-12)


def test_deann_k_equals_n_large_is_naive():
    X = np.random.default_rng(7).normal(size=(5000, 8)).astype(np.float32)
    q = np.random.default_rng(8).normal(size=8)
    ds, od = g.Dataset.from_array(X), O.Data(X)
    for fam, h in [("gaussian", 1.2), ("exponential", 1.5), ("laplacian", 4.0)]:
        est = g.deann(ds, g.KernelSpec(fam, h), g.BruteForceIndex(ds), q, 5000, 0)
        ref = O.naive_kde(od, fam, h, q.reshape(1, -1))[0]
        assert est.value == pytest.approx(ref, rel=1e-12)


@pytest.mark.parametrize("family,h", [("gaussian", 2.0), ("exponential", 2.5), ("laplacian", 6.0)])
def test_deann_long_exclusion_list_matches_oracle(family, h):
    # k = 17000 > the 16384-entry shared-memory sort: CUB segmented sort path
    n, k, m, seed = 24_000, 17_000, 400, 2024
    X = np.random.default_rng(9).normal(size=(n, 8)).astype(np.float32)
    Q = np.random.default_rng(10).normal(size=(3, 8))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    vals, nbr, smp = g.deann_arrays(ds, g.KernelSpec(family, h), Q, k, m, seed=seed, export_neighbors=True,
                                    export_samples=True)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], k)
        np.testing.assert_array_equal(nbr[j], ri)
        assert not np.isin(smp[j], ri).any()
        ref = O.deann(od, family, h, NeighborReplay(ri, rd), Q[j], k, m, rng=IndexReplay(seed, j, n))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-12)


def test_black_box_index_long_exclusion_list():
    # a user index returning 20000 ids: dk_sample sorts them with the segmented sort
    n, k, m = 30_000, 20_000, 300
    X = np.random.default_rng(11).normal(size=(n, 5)).astype(np.float32)
    q = np.random.default_rng(12).normal(size=5)
    od = O.Data(X)
    ri, rd = O.brute_force_knn(od, q, k)

    class Fixed(g.AnnIndex):
        def query(self, y, kk):
            return g.NeighborList(ri, rd)  # ids in distance order, unsorted by id

    ds = g.Dataset.from_array(X)
    est = g.deann(ds, g.KernelSpec("gaussian", 1.7), Fixed(), q, k, m, rng=g.PhiloxSampler(99))
    ref = O.deann(od, "gaussian", 1.7, NeighborReplay(ri, rd), q, k, m,
                  rng=IndexReplay(99, 0, n))[0]
    assert est.neighbors_used == k
    assert est.value == pytest.approx(ref, rel=1e-12)


def test_deannp_long_exclusion_list_matches_oracle():
    n, k, m = 24_000, 17_000, 500
    X = np.random.default_rng(14).normal(size=(n, 6)).astype(np.float32)
    Q = np.random.default_rng(15).normal(size=(3, 6))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    st = g.RspState.from_dataset(ds, 8, cursor=23_500)
    got = g.deann_batch(ds, g.KernelSpec("exponential", 2.0), g.BruteForceIndex(ds), Q, k, m, rsp_state=st)
    ost = O.Permuted(od, 8, cursor=23_500)
    nb = lambda y, kk: O.brute_force_knn(od, y, kk)  # noqa: E731
    for j, q in enumerate(Q):
        ref = O.deann_rsp(od, "exponential", 2.0, nb, q, k, m, ost)
        assert got[j].value == pytest.approx(ref[0], rel=1e-12)
    assert st.cursor == ost.cursor
