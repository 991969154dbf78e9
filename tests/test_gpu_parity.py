"""GPU parity: every path through the C-ABI against the oracle / reference goldens.

Tolerances (BASELINE.json north_star):
  exact KDE            <= 1e-4 relative vs the fp64 oracle; asserted at 1e-5
                       here.  The fused tile computes d2 = |q|^2+|x|^2-2S in
                       fp32, so a term's relative error is ~eps32*(|q|^2+|x|^2)/(2h^2):
                       3e-7 on the BASELINE configs, ~2e-6 on the reference's
                       small-h random acceptance instances.
  k-NN                 index sets identical up to ties within 1e-6 relative
                       (the cases here have no near-ties: identical sets+order)
  RS / DEANN           <= 1e-5 relative given the same sample indices (the GPU
                       computes these in fp64: we assert 1e-12)
"""

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
    return float(np.max(np.abs(a - b) / np.abs(b)))


# ------------------------------------------------------------------ exact KDE


def test_naive_goldens(golden):
    for i in golden["naive_cases"]:
        X, Q, v = golden[f"naive_{i}_X"], golden[f"naive_{i}_Q"], golden[f"naive_{i}_v"]
        h, fi = golden[f"naive_{i}_meta"]
        got = g.naive_kde(g.Dataset.from_array(X), g.KernelSpec(FAMILIES[int(fi)], float(h)), Q).values
        assert _rel(got, v) < KDE_RTOL, (i, FAMILIES[int(fi)])


def test_acceptance1_twenty_instances(golden):
    worst = 0.0
    for i in range(20):
        X, q = golden[f"acc1_{i}_X"], golden[f"acc1_{i}_q"]
        v, h, fi = golden[f"acc1_{i}_v"]
        got = g.naive_kde(g.Dataset.from_array(X), g.KernelSpec(FAMILIES[int(fi)], float(h)), q.reshape(1, -1))
        worst = max(worst, abs(got.values[0] - v) / v)
        assert got.kernel_evals == X.shape[0]
    assert worst < KDE_RTOL


def test_naive_two_copies_is_one():
    y = np.array([1.5, -2.0], dtype=np.float32)
    ds = g.Dataset.from_array(np.vstack([y, y]))
    out = g.naive_kde(ds, g.KernelSpec("gaussian", 1.0), y.reshape(1, -1))
    assert out.values[0] == pytest.approx(1.0, rel=1e-7)
    assert out.kernel_evals == 2


def test_naive_half_mass_when_far_point_underflows():
    y = np.zeros(2, dtype=np.float32)
    far = np.full(2, 1e6, dtype=np.float32)
    ds = g.Dataset.from_array(np.vstack([y, far]))
    for fam in FAMILIES:
        assert g.naive_kde(ds, g.KernelSpec(fam, 1.0), y.reshape(1, -1)).values[0] == pytest.approx(0.5, rel=1e-7)


@pytest.mark.parametrize("family,h", [("gaussian", 300.0), ("exponential", 400.0), ("laplacian", 4000.0)])
def test_naive_integer_rows_exact_mode(family, h):
    rng = np.random.default_rng(1)
    X = rng.integers(0, 256, size=(3001, 128)).astype(np.float32)   # ragged n
    Q = rng.integers(0, 256, size=(131, 128)).astype(np.float64)     # ragged nq
    ds = g.Dataset.from_array(X)
    assert ds.exact_mode
    got = g.naive_kde(ds, g.KernelSpec(family, h), Q).values
    assert _rel(got, O.naive_kde(O.Data(X), family, h, Q)) < KDE_RTOL


def test_naive_integer_rows_fractional_queries_switch_to_split():
    rng = np.random.default_rng(2)
    X = rng.integers(0, 50, size=(2000, 40)).astype(np.float32)
    Q = rng.integers(0, 50, size=(20, 40)) + 0.37
    ds = g.Dataset.from_array(X)
    got = g.naive_kde(ds, g.KernelSpec("gaussian", 15.0), Q).values
    assert _rel(got, O.naive_kde(O.Data(X), "gaussian", 15.0, Q)) < KDE_RTOL


@pytest.mark.parametrize("n,d,nq", [(1, 1, 1), (255, 3, 7), (257, 64, 129), (5000, 65, 300), (700, 200, 33)])
def test_naive_ragged_shapes(n, d, nq):
    rng = np.random.default_rng(n + d)
    X = rng.normal(size=(n, d)).astype(np.float32) + 3.0   # offset: exercises centring
    Q = rng.normal(size=(nq, d)) + 3.0
    h = math.sqrt(d)
    ds = g.Dataset.from_array(X)
    for fam in FAMILIES:
        got = g.naive_kde(ds, g.KernelSpec(fam, h if fam != "laplacian" else 2 * d ** 0.75), Q).values
        ref = O.naive_kde(O.Data(X), fam, h if fam != "laplacian" else 2 * d ** 0.75, Q)
        assert _rel(got, ref) < KDE_RTOL, fam


def test_naive_empty_query_batch():
    ds = g.Dataset.from_array(np.ones((4, 3), dtype=np.float32))
    assert g.naive_kde(ds, g.KernelSpec("gaussian", 1.0), np.zeros((0, 3))).values.shape == (0,)


def test_naive_dimension_mismatch():
    ds = g.Dataset.from_array(np.ones((10, 3), dtype=np.float32))
    with pytest.raises(ValueError):
        g.naive_kde(ds, g.KernelSpec("gaussian", 1.0), np.zeros((1, 4)))


def test_nonfinite_dataset_rejected():
    X = np.ones((5, 2), dtype=np.float32)
    X[3, 1] = np.nan
    with pytest.raises(ValueError, match="finite"):
        g.Dataset.from_array(X)


def test_reference_dataset_objects_are_accepted():
    class RefLike:
        def __init__(self, data):
            self.data = data

    X = np.random.default_rng(3).normal(size=(300, 5)).astype(np.float32)
    q = np.random.default_rng(4).normal(size=(2, 5))
    got = g.naive_kde(RefLike(X), g.KernelSpec("exponential", 1.0), q).values
    assert _rel(got, O.naive_kde(O.Data(X), "exponential", 1.0, q)) < KDE_RTOL


def test_sq_norms_and_kernel_values():
    X = np.random.default_rng(5).normal(size=(100, 7)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    np.testing.assert_allclose(ds.sq_norms, O.Data(X).sq_norms, rtol=1e-15)
    d = np.array([0.0, 1.0, 2.5, 1e4])
    for fam in FAMILIES:
        np.testing.assert_allclose(g.kernel_from_distance(g.KernelSpec(fam, 1.3), d),
                                   O.kernel_from_distance(fam, 1.3, d), rtol=1e-15)
    assert g.kernel_from_distance(g.KernelSpec("gaussian", 0.5), 3.0) == pytest.approx(math.exp(-6.0), rel=1e-14)
    with pytest.raises(ValueError):
        g.kernel_from_distance(g.KernelSpec("gaussian", 1.0), -1.0)


# ------------------------------------------------------------------ k-NN


def test_knn_golden_with_ties(golden):
    ds = g.Dataset.from_array(golden["knn_X"])
    idx, d2 = g.knn_batch(ds, golden["knn_Q"], 25)
    np.testing.assert_array_equal(idx, golden["knn_idx"])
    np.testing.assert_allclose(d2, golden["knn_d2"], rtol=1e-6, atol=1e-9)


def test_knn_hand_geometry_and_tie_break():
    ds = g.Dataset.from_array(np.array([[0, 0], [1, 0], [5, 0]], dtype=np.float32))
    assert g.brute_force_knn(ds, [0.9, 0.0], 2).indices.tolist() == [1, 0]
    ds = g.Dataset.from_array(np.zeros((3, 2), dtype=np.float32))
    assert g.brute_force_knn(ds, [1.0, 0.0], 2).indices.tolist() == [0, 1]


def test_knn_full_sort_oracle_and_k_equals_n():
    rng = np.random.default_rng(1)
    X = rng.normal(size=(200, 8)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    od = O.Data(X)
    for _ in range(5):
        q = rng.normal(size=8)
        d2 = ((X.astype(np.float64) - q) ** 2).sum(axis=1)
        order = np.lexsort((np.arange(200), d2))
        for k in (1, 7, 50, 200):
            nl = g.brute_force_knn(ds, q, k)
            assert nl.indices.tolist() == order[:k].tolist()
            ri, rd = O.brute_force_knn(od, q, k)
            np.testing.assert_allclose(nl.sq_distances, rd, rtol=1e-6, atol=1e-12)


def test_knn_large_n_matches_oracle():
    rng = np.random.default_rng(9)
    centers = rng.normal(scale=3.0, size=(20, 24))
    X = (centers[rng.integers(0, 20, 60_000)] + rng.normal(size=(60_000, 24))).astype(np.float32)
    Q = centers[rng.integers(0, 20, 40)] + rng.normal(size=(40, 24))
    ds = g.Dataset.from_array(X)
    od = O.Data(X)
    idx, d2 = g.knn_batch(ds, Q, 100)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], 100)
        np.testing.assert_array_equal(idx[j], ri)
        np.testing.assert_allclose(d2[j], rd, rtol=1e-6)


def test_knn_many_duplicates_fallback_path():
    # 3000 identical rows: the approximate certificate cannot separate them,
    # the exact fallback must still return the lowest indices
    X = np.zeros((6000, 4), dtype=np.float32)
    X[3000:] = np.random.default_rng(2).normal(size=(3000, 4)) + 10
    ds = g.Dataset.from_array(X)
    idx, d2 = g.knn_batch(ds, np.zeros((3, 4)), 64)
    assert (idx == np.arange(64)).all()
    assert (d2 == 0).all()


def test_knn_small_dataset_selects_without_exact_fallback(monkeypatch):
    # n <= 8192: every row is a candidate (tau = inf); the rows past n in the last tile
    # must not be appended, or every query overflows into the exact-scan fallback
    import ctypes

    from paper_2107_02736_b200 import _lib

    monkeypatch.setenv("DK_KNN_STATS", "1")
    X = np.random.default_rng(8).normal(size=(3001, 24)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    Q = np.random.default_rng(9).normal(size=(40, 24))
    idx, _ = g.knn_batch(ds, Q, 17)
    od = O.Data(X)
    for j in range(len(Q)):
        np.testing.assert_array_equal(idx[j], O.brute_force_knn(od, Q[j], 17)[0])
    v = [ctypes.c_int64() for _ in range(4)]
    _lib.check(_lib.load().dk_knn_stats(ds.handle, *[ctypes.byref(x) for x in v]))
    queries, cand_sum, _, fallbacks = (x.value for x in v)
    assert queries == len(Q) and fallbacks == 0
    assert cand_sum == len(Q) * X.shape[0]


def test_knn_pruned_path_clustered_ties_and_far_queries():
    # >= 512 tiles: the FILTER pass runs over k-means balls (capi.cu knn_device, pruned);
    # duplicated rows (ties across balls), queries on data points, between clusters and far
    # outside every ball must all give the brute-force answer (ann.py:82-102 tie rule)
    rng = np.random.default_rng(21)
    cent = rng.normal(0.0, 4.0, size=(40, 24))
    lab = rng.integers(0, 40, size=300_000)
    X = (cent[lab] + rng.normal(0.0, 1.0, size=(300_000, 24))).astype(np.float32)
    X[250_000:250_500] = X[1000:1500]  # exact duplicates far apart in row order
    ds = g.Dataset.from_array(X)
    Q = np.concatenate([
        X[[1000, 1001, 77, 299_999]].astype(np.float64),                 # on data points (ties)
        0.5 * (cent[:6] + cent[6:12]),                                   # between clusters
        rng.normal(0.0, 40.0, size=(4, 24)),                             # far outside every ball
        cent[lab[:6]] + rng.normal(0.0, 1.0, size=(6, 24)),             # ordinary
    ])
    idx, d2 = g.knn_batch(ds, Q, 30)
    od = O.Data(X)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], 30)
        np.testing.assert_array_equal(idx[j], ri)
        np.testing.assert_allclose(d2[j], rd, rtol=1e-9, atol=1e-12)


def test_knn_out_of_range():
    ds = g.Dataset.from_array(np.random.default_rng(0).normal(size=(5, 2)).astype(np.float32))
    for bad in (0, 6):
        with pytest.raises(ValueError):
            g.brute_force_knn(ds, np.zeros(2), bad)


def test_returned_distances_match_recomputation():
    X = np.random.default_rng(6).normal(size=(80, 5)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    q = np.random.default_rng(7).normal(size=5)
    nl = g.brute_force_knn(ds, q, 9)
    for i, dd in zip(nl.indices, nl.sq_distances):
        ref = float(((X[i].astype(np.float64) - q) ** 2).sum())
        assert dd == pytest.approx(ref, rel=1e-6, abs=1e-12)


# ------------------------------------------------------------------ sampling / DEANN


def test_rs_and_deann_goldens_under_replayed_stream(golden):
    """Reference (deann.rs_kde / deann.deann, fed the GPU's Philox stream) vs GPU."""
    X, Q = golden["samp_X"], golden["samp_Q"]
    seed = int(golden["samp_seed"][0])
    ds = g.Dataset.from_array(X)
    it_rs, it_de = iter(golden["samp_rs"]), iter(golden["samp_deann"])
    for j, q in enumerate(Q):
        for fam, h in [("gaussian", 1.3), ("exponential", 1.1), ("laplacian", 2.5)]:
            spec = g.KernelSpec(fam, h)
            est = g.rs_kde(ds, spec, q, 37, g.PhiloxSampler(seed, position=j))
            assert est.value == pytest.approx(next(it_rs), rel=1e-12)
            assert est.kernel_evals == est.samples_used == 37
            v, nbr, _ = g.deann_arrays(ds, spec, q.reshape(1, -1), 15, 50, seed=seed + 1, query_base=j,
                                       export_neighbors=True)
            assert v[0] == pytest.approx(next(it_de), rel=1e-12)
        np.testing.assert_array_equal(nbr[0], golden["samp_nbr"][j])


@pytest.mark.parametrize("family", FAMILIES)
def test_deann_batch_replay_parity(family):
    rng = np.random.default_rng(11)
    X = rng.normal(size=(5000, 12)).astype(np.float32)
    Q = rng.normal(size=(64, 12))
    h = {"gaussian": 1.5, "exponential": 1.2, "laplacian": 4.0}[family]
    ds = g.Dataset.from_array(X)
    od = O.Data(X)
    k, m, seed = 40, 300, 987654321
    vals, nbr, smp = g.deann_arrays(ds, g.KernelSpec(family, h), Q, k, m, seed=seed, export_neighbors=True,
                                    export_samples=True)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], k)
        np.testing.assert_array_equal(nbr[j], ri)
        excl = set(ri.tolist())
        assert not (set(smp[j].tolist()) & excl)
        ref = O.deann(od, family, h, NeighborReplay(ri, rd), Q[j], k, m, rng=IndexReplay(seed, j, X.shape[0]))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-12)


def test_exported_samples_are_the_first_m_accepted():
    from oracle.philox import draws

    X = np.random.default_rng(12).normal(size=(300, 4)).astype(np.float32)
    q = np.zeros((1, 4))
    ds = g.Dataset.from_array(X)
    _, nbr, smp = g.deann_arrays(ds, g.KernelSpec("gaussian", 1.0), q, 30, 200, seed=5, export_neighbors=True,
                                 export_samples=True)
    stream = draws(5, 0, 0, 5000, 300)
    keep = stream[~np.isin(stream, nbr[0])][:200]
    np.testing.assert_array_equal(smp[0], keep)


def test_deann_k_zero_equals_rs_exactly():
    X = np.random.default_rng(21).normal(size=(70, 4)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    kernel = g.KernelSpec("exponential", 1.2)
    q = np.random.default_rng(22).normal(size=4)
    a = g.deann(ds, kernel, None, q, 0, 25, rng=np.random.default_rng(77))
    b = g.rs_kde(ds, kernel, q, 25, np.random.default_rng(77))
    assert a.value == b.value


def test_deann_k_equals_n_is_naive(golden):
    X, q = golden["lim_X"], golden["lim_q"]
    ds = g.Dataset.from_array(X)
    est = g.deann(ds, g.KernelSpec("gaussian", 1.4), g.BruteForceIndex(ds), q, 80, 0)
    assert est.value == pytest.approx(golden["lim_naive"][0], rel=1e-12)
    assert est.neighbors_used == 80 and est.samples_used == 0 and not est.truncated


def test_deann_truncated_flag_and_costs():
    X = np.random.default_rng(19).normal(size=(40, 3)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    est = g.deann(ds, g.KernelSpec("gaussian", 1.0), g.BruteForceIndex(ds), np.zeros(3), 5, 0)
    assert est.truncated and est.kernel_evals == 5
    rng = np.random.default_rng(0)
    for k in (0, 1, 10, 39):
        for m in (0, 1, 60):
            if m > 0 and k >= 40:
                continue
            e = g.deann(ds, g.KernelSpec("exponential", 1.0), g.BruteForceIndex(ds),
                        rng.normal(size=3), k, m, rng=np.random.default_rng(k + m) if m else None)
            assert e.kernel_evals == e.neighbors_used + e.samples_used
            assert 0.0 <= e.value <= 1.0 + 1e-12


def test_deann_parameter_validation():
    ds = g.Dataset.from_array(np.random.default_rng(33).normal(size=(20, 2)).astype(np.float32))
    kernel = g.KernelSpec("gaussian", 1.0)
    bf = g.BruteForceIndex(ds)
    rng = np.random.default_rng(0)
    with pytest.raises(ValueError):
        g.deann(ds, kernel, bf, np.zeros(2), 21, 0)
    with pytest.raises(ValueError):
        g.deann(ds, kernel, bf, np.zeros(2), 20, 5, rng=rng)
    with pytest.raises(ValueError):
        g.deann(ds, kernel, bf, np.zeros(2), 2, -1, rng=rng)
    with pytest.raises(ValueError):
        g.deann(ds, kernel, bf, np.zeros(2), 2, 5)
    with pytest.raises(ValueError):
        g.deann(ds, kernel, bf, np.zeros(3), 2, 5, rng=rng)
    with pytest.raises(ValueError):
        g.rs_kde(ds, kernel, np.zeros(2), 0, rng)


def test_black_box_ann_path_matches_oracle():
    """A non-GPU AnnIndex (fixed neighbour list, cf. test_acceptance.py:60-68)."""
    X = np.random.default_rng(40).normal(size=(500, 6)).astype(np.float32)
    q = np.random.default_rng(41).normal(size=6)
    od = O.Data(X)
    ri, rd = O.brute_force_knn(od, q, 20)
    sub_i, sub_d = ri[::2], rd[::2]    # a deliberately poor (recall 0.5) index

    class Fixed(g.AnnIndex):
        def query(self, y, k):
            return g.NeighborList(sub_i, sub_d)

    ds = g.Dataset.from_array(X)
    for fam, h in [("gaussian", 1.3), ("laplacian", 3.0)]:
        est = g.deann(ds, g.KernelSpec(fam, h), Fixed(), q, 20, 80, rng=g.PhiloxSampler(55))
        ref = O.deann(od, fam, h, NeighborReplay(sub_i, sub_d), q, 20, 80, rng=IndexReplay(55, 0, 500))[0]
        assert est.neighbors_used == 10
        assert est.value == pytest.approx(ref, rel=1e-12)


def test_rs_unbiased_smoke():
    X = np.random.default_rng(7).normal(size=(100, 3)).astype(np.float32)
    q = np.random.default_rng(8).normal(size=3)
    ds = g.Dataset.from_array(X)
    kernel = g.KernelSpec("exponential", 1.5)
    exact = O.naive_kde(O.Data(X), "exponential", 1.5, q.reshape(1, -1))[0]
    trials, _, _ = g.deann_arrays(ds, kernel, np.tile(q, (8000, 1)), 0, 8, seed=1234)
    se = trials.std(ddof=1) / math.sqrt(len(trials))
    assert abs(trials.mean() - exact) < 4 * se


def test_deann_unbiased_smoke_exact_neighbors():
    rng = np.random.default_rng(31)
    centers = rng.normal(scale=12.0, size=(5, 3))
    X = (centers[np.arange(200) % 5] + rng.normal(size=(200, 3))).astype(np.float32)
    q = centers[0] + rng.normal(size=3)
    ds = g.Dataset.from_array(X)
    kernel = g.KernelSpec("exponential", 2.0)
    exact = O.naive_kde(O.Data(X), "exponential", 2.0, q.reshape(1, -1))[0]
    trials, _, _ = g.deann_arrays(ds, kernel, np.tile(q, (8000, 1)), 10, 20, seed=32)
    se = trials.std(ddof=1) / math.sqrt(len(trials))
    assert abs(trials.mean() - exact) < 4 * se


def test_deann_batch_list_api():
    X = np.random.default_rng(37).normal(size=(50, 3)).astype(np.float32)
    Q = np.random.default_rng(38).normal(size=(4, 3))
    ds = g.Dataset.from_array(X)
    out = g.deann_batch(ds, g.KernelSpec("exponential", 1.0), g.BruteForceIndex(ds), Q, 5, 10,
                        rng=np.random.default_rng(3))
    assert len(out) == 4 and all(e.neighbors_used == 5 and e.samples_used == 10 for e in out)


def test_fit_bandwidth_hits_target_median():
    from paper_2107_02736_b200 import fit_bandwidth

    rng = np.random.default_rng(0)
    X = rng.normal(size=(4000, 8)).astype(np.float32)
    P = rng.normal(size=(200, 8))
    h = fit_bandwidth(g.Dataset.from_array(X), P, "gaussian", 1e-2, rel_tol=0.01)
    vals = O.naive_kde(O.Data(X), "gaussian", h, P)
    med = float(np.sort(vals)[(len(vals) - 1) // 2])
    assert abs(med - 1e-2) <= 0.0101 * 1e-2


class _BlackBoxExact(g.AnnIndex):
    """A user index that is NOT recognised as the GPU brute force (black-box path)."""

    def __init__(self, ds):
        self.ds = ds

    def query(self, query, k):
        return g.brute_force_knn(self.ds, query, k)


@pytest.mark.parametrize("rng", [11, "philox"])
def test_deann_batch_black_box_index_uses_one_stream(rng):
    """a black-box index with an int seed must not restart the Philox stream per
    query; the per-query loop equals the fused brute-force batch value for value."""
    X = np.random.default_rng(41).normal(size=(300, 5)).astype(np.float32)
    Q = np.random.default_rng(42).normal(size=(6, 5))
    ds = g.Dataset.from_array(X)
    spec = g.KernelSpec("gaussian", 1.3)
    mk = (lambda: 11) if rng == 11 else (lambda: g.PhiloxSampler(11))
    fused = g.deann_batch(ds, spec, g.BruteForceIndex(ds), Q, 7, 40, rng=mk())
    loop = g.deann_batch(ds, spec, _BlackBoxExact(ds), Q, 7, 40, rng=mk())
    a = np.array([e.value for e in fused])
    b = np.array([e.value for e in loop])
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    assert len(set(np.round(b, 12))) == len(b)  # distinct queries, distinct streams


def _oracle_knn_block(od, Q, k, step=200):
    """O.brute_force_knn for many queries (the reference's batch_sqdist + _smallest_k per row)."""
    out_i = np.empty((len(Q), k), dtype=np.int64)
    ids = np.arange(od.n, dtype=np.int64)
    for lo in range(0, len(Q), step):
        D = O.batch_sqdist(Q[lo:lo + step], od.x64, od.sq_norms)
        for r in range(D.shape[0]):
            out_i[lo + r] = O.smallest_k(D[r], ids, k)[0]
    return out_i


@pytest.fixture(scope="module")
def clustered_150k():
    rng = np.random.default_rng(77)
    centers = rng.normal(scale=6.0, size=(300, 32))
    lab = rng.integers(0, 300, size=150_000)
    X = (centers[lab] + rng.normal(size=(150_000, 32))).astype(np.float32)
    qlab = rng.integers(0, 300, size=2000)
    Q = centers[qlab] + rng.normal(size=(2000, 32))
    Q[:20] = X[rng.integers(0, len(X), 20)]            # on-point queries (distance-0 neighbour)
    Q[20:40] = rng.normal(scale=40.0, size=(20, 32))    # far from every cluster
    return X, Q, g.Dataset.from_array(X), O.Data(X)


def test_pruned_knn_many_queries_exact(clustered_150k, monkeypatch):
    """the pruned FILTER path (>= 512 tiles) on 2,000 queries spread over many balls,
    compared query by query with the reference's brute force; then again split into 4 batches
    (DK_KNN_MAX_BATCH test hook: multi-batch qperm scatter and per-batch unit plans), with the
    bitonic tau path (DK_TAU_SORT) and with the near-tile threshold lists (DK_KNN_HOME) — all
    identical, indices and distances."""
    X, Q, ds, od = clustered_150k
    k = 50
    idx, d2 = g.knn_batch(ds, Q, k)
    want = _oracle_knn_block(od, Q, k)
    np.testing.assert_array_equal(idx, want)
    monkeypatch.setenv("DK_KNN_MAX_BATCH", "512")
    idx2, d22 = g.knn_batch(ds, Q, k)
    monkeypatch.delenv("DK_KNN_MAX_BATCH")
    monkeypatch.setenv("DK_TAU_SORT", "1")
    idx3, d23 = g.knn_batch(ds, Q, k)
    monkeypatch.delenv("DK_TAU_SORT")
    monkeypatch.setenv("DK_KNN_HOME", "1")  # threshold from per-block near-tile lists
    idx4, d24 = g.knn_batch(ds, Q, k)
    monkeypatch.delenv("DK_KNN_HOME")
    for a, b in ((idx2, d22), (idx3, d23), (idx4, d24)):
        np.testing.assert_array_equal(a, idx)
        np.testing.assert_array_equal(b, d2)


def test_merge_topk_matches_single_shard(clustered_150k):
    """dk_merge_topk (warp per query) of 3 row shards' exact top-k equals the whole dataset's."""
    import torch

    X, Q, ds, od = clustered_150k
    k = 40
    Qs = Q[:300]
    full_i, full_d = g.knn_batch(ds, Qs, k)
    cuts = [0, 41_000, 97_777, len(X)]
    parts_i, parts_d = [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        sh = g.Dataset.from_array(X[a:b], global_offset=a, global_n=len(X))
        i, d = g.knn_batch(sh, Qs, k)
        parts_i.append(i)
        parts_d.append(d)
    from paper_2107_02736_b200.sharded import GpuShardEngine

    eng = GpuShardEngine(None, global_offset=0, global_n=len(X), dataset=ds)
    mi, md = eng.merge_topk(torch.as_tensor(np.stack(parts_i), device="cuda"),
                            torch.as_tensor(np.stack(parts_d), device="cuda"), k)
    np.testing.assert_array_equal(mi.cpu().numpy(), full_i)
    np.testing.assert_array_equal(md.cpu().numpy(), full_d)
