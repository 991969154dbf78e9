"""GPU inverted-file index against the reference goldens and the oracle.

Goldens come from the real reference (tests/golden/make_golden.py: ivf_build,
ivf_query, IvfAnnIndex.query, save_ivf_index); the reference's own tests
(test_ann.py:74-188, acceptance 7 at test_acceptance.py:260-285) are restated
here against the GPU implementation.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2107_02736_b200 as g
from oracle import deann_oracle as O
from oracle.philox import IndexReplay, NeighborReplay

pytestmark = pytest.mark.gpu

CASES = [("ivf_a", 500, 6, 12, 3), ("ivf_b", 20_000, 16, 64, 7)]


def _data(n, d, seed):
    X = np.random.default_rng(seed).normal(size=(n, d)).astype(np.float32)
    Q = np.random.default_rng(seed + 1).normal(size=(8, d))
    return X, Q


@pytest.mark.parametrize("tag,n,d,C,seed", CASES)
def test_build_matches_reference(golden, tag, n, d, C, seed):
    X, _ = _data(n, d, seed)
    index = g.ivf_build(g.Dataset.from_array(X), C, seed)
    np.testing.assert_allclose(index.centroids, golden[f"{tag}_cent"], rtol=1e-12, atol=1e-15)
    rows, off = golden[f"{tag}_rows"], golden[f"{tag}_off"]
    for c in range(C):
        np.testing.assert_array_equal(index.assignments[c], rows[off[c]:off[c + 1]])
    assert index.seed == seed and index.n_clusters == C and index.d == d


@pytest.mark.parametrize("tag,n,d,C,seed", CASES)
def test_queries_match_reference(golden, tag, n, d, C, seed):
    X, Q = _data(n, d, seed)
    ds = g.Dataset.from_array(X)
    index = g.ivf_build(ds, C, seed)
    i = 0
    for p in golden[f"{tag}_probes"]:
        p = int(p)
        ann = g.IvfAnnIndex(ds, index, p)
        bi, bd, bc = g.ivf_query_batch(index, ds, Q, 10, p)
        for j, q in enumerate(Q):
            gi, gd = golden[f"{tag}_q_idx"][i], golden[f"{tag}_q_d2"][i]
            nl = g.ivf_query(index, ds, q, 10, p)
            np.testing.assert_array_equal(nl.indices, gi[gi >= 0])
            np.testing.assert_allclose(nl.sq_distances, gd[gi >= 0], rtol=1e-12)
            assert bc[j] == len(nl) and (bi[j, :bc[j]] == nl.indices).all()
            gi, gd = golden[f"{tag}_ann_idx"][i], golden[f"{tag}_ann_d2"][i]
            nl = ann.query(q, 10)
            np.testing.assert_array_equal(nl.indices, gi[gi >= 0])
            np.testing.assert_allclose(nl.sq_distances, gd[gi >= 0], rtol=1e-12)
            i += 1


def test_reference_index_objects_and_files(golden, tmp_path):
    tag, n, d, C, seed = CASES[0]
    X, Q = _data(n, d, seed)
    ds = g.Dataset.from_array(X)
    p = tmp_path / "ref.ivf"
    p.write_bytes(golden["ivf_a_file"].tobytes())
    loaded = g.load_ivf_index(p)  # the reference's own file
    np.testing.assert_array_equal(loaded.centroids, golden[f"{tag}_cent"])
    built = g.ivf_build(ds, C, seed)
    out = tmp_path / "ours.ivf"
    g.save_ivf_index(built, out)
    assert out.read_bytes() == p.read_bytes()  # byte-identical container
    for q in Q:
        a = g.ivf_query(loaded, ds, q, 10, 3)
        b = g.ivf_query(built, ds, q, 10, 3)
        assert a.indices.tolist() == b.indices.tolist()
    with pytest.raises(ValueError):
        bad = tmp_path / "bad.ivf"
        bad.write_bytes(b"NOTANIVF" + bytes(20))
        g.load_ivf_index(bad)


def test_full_probe_equals_brute_force_acceptance7():
    # test_acceptance.py:260-285 restated: full probe == brute force, recall monotone in n_probe
    rng = np.random.default_rng(707)
    for trial in range(50):
        n = int(rng.integers(50, 301))
        d = int(rng.integers(2, 9))
        X = rng.normal(size=(n, d)).astype(np.float32)
        ds = g.Dataset.from_array(X)
        C = int(rng.integers(2, min(13, n)))
        index = g.ivf_build(ds, C, seed=trial)
        q = rng.normal(size=d)
        k = int(rng.integers(1, min(20, n) + 1))
        exact = g.brute_force_knn(ds, q, k)
        assert g.ivf_query(index, ds, q, k, C).indices.tolist() == exact.indices.tolist()
        rec = [g.recall(g.ivf_query(index, ds, q, k, p), exact) for p in range(1, C + 1)]
        assert all(b >= a for a, b in zip(rec, rec[1:]))
        cent, lists = O.ivf_build(O.Data(X), C, trial)
        np.testing.assert_allclose(index.centroids, cent, rtol=1e-12, atol=1e-15)
        assert all((a == b).all() for a, b in zip(index.assignments, lists))


def test_reference_unit_cases():
    # test_ann.py:74-153
    X = np.random.default_rng(3).normal(size=(40, 3)).astype(np.float32)
    idx = g.ivf_build(g.Dataset.from_array(X), 1, seed=0)
    assert sorted(idx.assignments[0].tolist()) == list(range(40))
    np.testing.assert_allclose(idx.centroids[0], X.astype(np.float64).mean(axis=0), rtol=1e-9)
    rng = np.random.default_rng(5)
    two = np.concatenate([rng.normal(size=(60, 4)) - 20, rng.normal(size=(60, 4)) + 20]).astype(np.float32)
    ds2 = g.Dataset.from_array(two)
    idx = g.ivf_build(ds2, 2, seed=5)
    sets = [set(a.tolist()) for a in idx.assignments]
    assert set(range(60)) in sets and set(range(60, 120)) in sets
    nl = g.ivf_query(idx, ds2, two[10].astype(np.float64) + 0.01, 20, 1)
    assert np.all(nl.indices < 60)
    short = g.ivf_query(idx, ds2, two[0].astype(np.float64), 80, 1)
    assert 0 < len(short) <= 60
    X12 = np.random.default_rng(7).normal(size=(12, 2)).astype(np.float32)
    idx = g.ivf_build(g.Dataset.from_array(X12), 12, seed=1)
    assert sorted(np.concatenate([a for a in idx.assignments if len(a)]).tolist()) == list(range(12))
    ds = g.Dataset.from_array(np.random.default_rng(0).normal(size=(10, 2)).astype(np.float32))
    for bad in (0, 11):
        with pytest.raises(ValueError):
            g.ivf_build(ds, bad, seed=0)
    ds30 = g.Dataset.from_array(np.random.default_rng(1).normal(size=(30, 3)).astype(np.float32))
    idx = g.ivf_build(ds30, 4, seed=0)
    for args in ((np.zeros(3), 0, 1), (np.zeros(3), 3, 0), (np.zeros(3), 3, 5), (np.zeros(4), 3, 2)):
        with pytest.raises(ValueError):
            g.ivf_query(idx, ds30, *args)
    a = g.ivf_build(ds30, 4, seed=9)
    b = g.ivf_build(ds30, 4, seed=9)
    np.testing.assert_array_equal(a.centroids, b.centroids)


def test_duplicate_rows_and_ties():
    # many identical rows: argmin ties to the lower centroid, scan ties to the lower row
    X = np.repeat(np.random.default_rng(8).integers(-2, 3, size=(40, 3)), 5, axis=0).astype(np.float32)
    ds = g.Dataset.from_array(X)
    index = g.ivf_build(ds, 6, seed=2)
    cent, lists = O.ivf_build(O.Data(X), 6, 2)
    np.testing.assert_allclose(index.centroids, cent, rtol=1e-12, atol=1e-15)
    assert all((a == b).all() for a, b in zip(index.assignments, lists))
    for q in X[:10].astype(np.float64):
        ri, rd = O.ivf_query(O.Data(X), cent, lists, q, 12, 3)
        nl = g.ivf_query(index, ds, q, 12, 3)
        np.testing.assert_array_equal(nl.indices, ri)


@pytest.mark.parametrize("family,h", [("gaussian", 1.2), ("exponential", 1.0), ("laplacian", 3.0)])
def test_deann_with_ivf_index_matches_oracle(family, h):
    n, d = 6000, 8
    X = np.random.default_rng(21).normal(size=(n, d)).astype(np.float32)
    Q = np.random.default_rng(22).normal(size=(12, d))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    ann = g.IvfAnnIndex.build(ds, 32, seed=4, n_probe=2)
    k, m, seed = 50, 300, 77
    batch = g.deann_batch(ds, g.KernelSpec(family, h), ann, Q, k, m, rng=g.PhiloxSampler(seed))
    cent, lists = O.ivf_build(od, 32, 4)
    for j, q in enumerate(Q):
        ri, rd = O.ivf_query(od, cent, lists, q, k, 2, formula=1)
        ref = O.deann(od, family, h, NeighborReplay(ri, rd), q, k, m, rng=IndexReplay(seed, j, n))
        assert batch[j].neighbors_used == len(ri)
        assert batch[j].value == pytest.approx(ref[0], rel=1e-12)
        one = g.deann(ds, g.KernelSpec(family, h), ann, q, k, m, rng=g.PhiloxSampler(seed, position=j))
        assert one.value == pytest.approx(batch[j].value, rel=1e-12)


def test_large_build_and_batch_scan_vs_oracle():
    n, d, C = 200_000, 24, 256
    rng = np.random.default_rng(31)
    centers = rng.normal(scale=4.0, size=(64, d))
    X = (centers[rng.integers(0, 64, n)] + rng.normal(size=(n, d))).astype(np.float32)
    Q = centers[rng.integers(0, 64, 64)] + rng.normal(size=(64, d))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    index = g.ivf_build(ds, C, seed=1)
    cent, lists = O.ivf_build(od, C, 1)
    np.testing.assert_allclose(index.centroids, cent, rtol=1e-10, atol=1e-12)
    same = sum((a.shape == b.shape and (a == b).all()) for a, b in zip(index.assignments, lists))
    assert same == C
    idx, d2, cnt = g.ivf_query_batch(index, ds, Q, 100, 8)
    for j in range(len(Q)):
        ri, rd = O.ivf_query(od, cent, lists, Q[j], 100, 8)
        np.testing.assert_array_equal(idx[j, :cnt[j]], ri)
        np.testing.assert_allclose(d2[j, :cnt[j]], rd, rtol=1e-12)


def test_large_k_beyond_the_shared_memory_top_k():
    # k > 4096: every probed candidate is sorted by (d2, row) on the device
    n, d = 30_000, 6
    X = np.random.default_rng(41).normal(size=(n, d)).astype(np.float32)
    X[:2000] = X[0]                                   # a block of exact ties
    Q = np.random.default_rng(42).normal(size=(3, d))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    index = g.ivf_build(ds, 16, seed=5)
    cent, lists = O.ivf_build(od, 16, 5)
    for q in np.vstack([Q, X[:1].astype(np.float64)]):
        for k, p in ((5000, 4), (30_000, 16)):
            nl = g.ivf_query(index, ds, q, k, p)
            ri, rd = O.ivf_query(od, cent, lists, q, k, p)
            np.testing.assert_array_equal(nl.indices, ri)
            np.testing.assert_allclose(nl.sq_distances, rd, rtol=1e-12, atol=1e-12)


def test_many_clusters_probe_by_segmented_sort():
    # n_clusters > 8192: the probe switches from the shared-memory sort to a radix sort
    rng = np.random.default_rng(43)
    n, d, C = 20_000, 4, 9000
    X = rng.normal(size=(n, d)).astype(np.float32)
    cent = X[rng.choice(n, C, replace=False)].astype(np.float64)
    cent[1] = cent[0]                                  # tied centroids: lower id first
    lab = np.empty(n, dtype=np.int64)
    for s in range(0, n, 2000):
        d2 = O.centroid_sqdists(X[s:s + 2000].astype(np.float64), O.Data(X[s:s + 2000]).sq_norms, cent)
        lab[s:s + 2000] = np.argmin(d2, axis=1)
    lists = [np.flatnonzero(lab == c).astype(np.int64) for c in range(C)]
    index = g.IvfIndex(centroids=cent, assignments=lists, seed=0)
    ds, od = g.Dataset.from_array(X), O.Data(X)
    Q = rng.normal(size=(5, d))
    for q in np.vstack([Q, cent[:1]]):
        for p in (1, 7, 40):
            nl = g.ivf_query(index, ds, q, 10, p)
            ri, rd = O.ivf_query(od, cent, lists, q, 10, p)
            np.testing.assert_array_equal(nl.indices, ri)
        ann = g.IvfAnnIndex(ds, index, 7)
        ri, _ = O.ivf_query(od, cent, lists, q, 10, 7, formula=1)
        np.testing.assert_array_equal(ann.query(q, 10).indices, ri)


@pytest.mark.parametrize("cap", [None, "1", "40"])
def test_two_phase_overflow_redo_for_far_queries(cap, monkeypatch):
    # queries far from every list pass many rows of the other probed lists under their phase-1
    # threshold; a candidate buffer that overflows (forced small with DK_IVF_CAP) sends the
    # query to the exact redo path
    if cap is not None:
        monkeypatch.setenv("DK_IVF_CAP", cap)
    rng = np.random.default_rng(47)
    n, d, C = 40_000, 12, 8
    X = rng.normal(size=(n, d)).astype(np.float32)
    Q = np.vstack([rng.normal(size=(6, d)), 60.0 * rng.normal(size=(6, d))])
    ds, od = g.Dataset.from_array(X), O.Data(X)
    index = g.ivf_build(ds, C, seed=3)
    cent, lists = O.ivf_build(od, C, 3)
    for k, p in ((10, 6), (100, 8)):
        idx, d2, cnt = g.ivf_query_batch(index, ds, Q, k, p)
        for j in range(len(Q)):
            ri, rd = O.ivf_query(od, cent, lists, Q[j], k, p)
            np.testing.assert_array_equal(idx[j, :cnt[j]], ri)
            np.testing.assert_allclose(d2[j, :cnt[j]], rd, rtol=1e-12)


@pytest.mark.parametrize("d", [13, 36])
def test_two_phase_odd_and_wide_rows(d):
    # row widths off the 16-byte copy path (13) and over several 16-dimension stages (36)
    rng = np.random.default_rng(53 + d)
    n, C = 30_000, 24
    centers = rng.normal(scale=3.0, size=(12, d))
    X = (centers[rng.integers(0, 12, n)] + rng.normal(size=(n, d))).astype(np.float32)
    Q = np.vstack([centers[rng.integers(0, 12, 20)] + rng.normal(size=(20, d)), 25.0 * rng.normal(size=(4, d))])
    ds, od = g.Dataset.from_array(X), O.Data(X)
    index = g.ivf_build(ds, C, seed=9)
    cent, lists = O.ivf_build(od, C, 9)
    for k, p in ((1, 3), (64, 7)):
        idx, d2, cnt = g.ivf_query_batch(index, ds, Q, k, p)
        for j in range(len(Q)):
            ri, rd = O.ivf_query(od, cent, lists, Q[j], k, p)
            np.testing.assert_array_equal(idx[j, :cnt[j]], ri)
            np.testing.assert_allclose(d2[j, :cnt[j]], rd, rtol=1e-12)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_arbitrary_lists_empty_lists_ties_and_short_probes(seed):
    # hand-made inverted lists (empty lists, lists shorter than k, duplicated rows across the
    # two phases), n_probe from 2 to C, k from 1 to beyond the probed rows; batch vs oracle
    rng = np.random.default_rng(300 + seed)
    n, d, C = int(rng.integers(40, 400)), int(rng.integers(1, 40)), int(rng.integers(3, 12))
    X = rng.normal(size=(n, d)).astype(np.float32)
    X[: n // 5] = X[0]                                   # a block of identical rows
    cent = rng.normal(size=(C, d))
    cent[1] = cent[0]                                     # tied centroids
    lab = rng.integers(0, C, n)
    lab[lab == C - 1] = 0                                 # list C-1 empty
    lists = [np.flatnonzero(lab == c).astype(np.int64) for c in range(C)]
    index = g.IvfIndex(centroids=cent, assignments=lists, seed=0)
    ds, od = g.Dataset.from_array(X), O.Data(X)
    Q = np.vstack([rng.normal(size=(7, d)), X[:2].astype(np.float64), 30.0 * rng.normal(size=(2, d))])
    for k, p in ((1, 2), (3, C), (int(rng.integers(5, 60)), max(2, C // 2)), (n, C)):
        idx, d2, cnt = g.ivf_query_batch(index, ds, Q, k, p)
        for j in range(len(Q)):
            ri, rd = O.ivf_query(od, cent, lists, Q[j], k, p)
            assert cnt[j] == len(ri)
            np.testing.assert_array_equal(idx[j, :cnt[j]], ri)
            np.testing.assert_allclose(d2[j, :cnt[j]], rd, rtol=1e-12, atol=1e-12)
            assert (idx[j, cnt[j]:] == -1).all()


@pytest.mark.parametrize("family,h,m", [("gaussian", 1.2, 0), ("laplacian", 3.0, 40), ("exponential", 1.0, 40)])
def test_deann_with_short_ivf_lists(family, h, m):
    # the probed lists hold fewer than k rows: k_hat < k neighbours, Z1 and the weights use k_hat
    n, d = 300, 6
    X = np.random.default_rng(61).normal(size=(n, d)).astype(np.float32)
    Q = np.random.default_rng(62).normal(size=(9, d))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    ann = g.IvfAnnIndex.build(ds, 32, seed=2, n_probe=1)
    k, seed = 50, 5
    batch = g.deann_batch(ds, g.KernelSpec(family, h), ann, Q, k, m, rng=g.PhiloxSampler(seed))
    cent, lists = O.ivf_build(od, 32, 2)
    for j, q in enumerate(Q):
        ri, rd = O.ivf_query(od, cent, lists, q, k, 1, formula=1)
        assert len(ri) < k
        ref = O.deann(od, family, h, NeighborReplay(ri, rd), q, k, m,
                      rng=IndexReplay(seed, j, n) if m else None)
        assert batch[j].neighbors_used == len(ri)
        assert batch[j].samples_used == m
        assert batch[j].value == pytest.approx(ref[0], rel=1e-12)


@pytest.mark.parametrize("tag", ["ivf_t1", "ivf_t2"])
def test_ivf_ann_index_fp32_ranking_near_ties(golden, tag):
    """IvfAnnIndex ranks the probed rows in fp32 by (key, probe position) before its fp64
    re-evaluation (ann.py:294-316).  On the engineered fp32 near-ties of the goldens (integer rows
    with |x|^2 > 2^24: fp32 keys collide for rows whose exact distances differ) the GPU equals the
    reference's own answers — batch and per-query calls — where exact ranking would not."""
    X, Q = golden[f"{tag}_X"], golden[f"{tag}_Q"]
    ds = g.Dataset.from_array(X)
    index = g.ivf_build(ds, len(golden[f"{tag}_cent"]), int(tag[-1]) + 10)
    rows, off = golden[f"{tag}_rows"], golden[f"{tag}_off"]
    for c in range(len(index.assignments)):
        np.testing.assert_array_equal(index.assignments[c], rows[off[c]:off[c + 1]])
    i = 0
    for p in golden[f"{tag}_probes"]:
        ann = g.IvfAnnIndex(ds, index, int(p))
        bi, bd, bc = ann.query_batch(Q, 10)
        for j, q in enumerate(Q):
            gi, gd = golden[f"{tag}_ann_idx"][i], golden[f"{tag}_ann_d2"][i]
            np.testing.assert_array_equal(bi[j, :bc[j]], gi[gi >= 0])
            np.testing.assert_array_equal(bd[j, :bc[j]], gd[gi >= 0])
            nl = ann.query(q, 10)
            np.testing.assert_array_equal(nl.indices, gi[gi >= 0])
            i += 1
