"""GPU parity at BASELINE.json's full configuration sizes.

Oracle comparisons use seeded query subsets (the fp64 oracle over 1e6+ rows is
seconds per query batch); size-independent properties cover the rest: the
partition-composition identity (Lemma 2, test_estimators.py:216-228), the
median-1e-3 bandwidth property on the pilot set, value ranges, and replayed
DEANN parity.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402
from dk_testutil import REPO  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from oracle.philox import IndexReplay, NeighborReplay  # noqa: E402

MAN = json.load(open(os.path.join(REPO, "tests", "golden", "bandwidths.json")))
KDE_RTOL = 1e-5  # gate: 1e-4


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b))))


@pytest.fixture(scope="module")
def c2():
    W = workloads.make("c2")
    return W, g.Dataset.from_array(W.X), O.Data(W.X)


@pytest.fixture(scope="module")
def c3():
    W = workloads.make("c3")
    return W, g.Dataset.from_array(W.X), O.Data(W.X)


def test_c2_naive_full_batch(c2):
    W, ds, od = c2
    h = MAN["c2"]["h"]
    assert ds.exact_mode  # integer rows: exact distance tiles
    vals = g.naive_kde(ds, g.KernelSpec("gaussian", h), W.Q).values
    assert vals.shape == (10_000,) and np.all(vals > 0) and np.all(vals <= 1)
    sel = np.random.default_rng(0).choice(10_000, 16, replace=False)
    assert _rel(vals[sel], O.naive_kde(od, "gaussian", h, W.Q[sel])) < KDE_RTOL
    # the bandwidth rule: lower median of the pilot KDE is 1e-3 within the 1% bisection tolerance
    pv = np.sort(g.naive_kde(ds, g.KernelSpec("gaussian", h), W.pilot).values)
    assert abs(pv[(len(pv) - 1) // 2] - 1e-3) <= 0.0101e-3


def test_c2_partition_composition(c2):
    W, ds, _ = c2
    h = MAN["c2"]["h"]
    kern = g.KernelSpec("gaussian", h)
    Q = W.Q[:512]
    full = g.naive_kde(ds, kern, Q).values
    cut = 377_777
    a = g.naive_kde(g.Dataset.from_array(W.X[:cut]), kern, Q).values
    b = g.naive_kde(g.Dataset.from_array(W.X[cut:]), kern, Q).values
    comb = (cut * a + (W.X.shape[0] - cut) * b) / W.X.shape[0]
    assert _rel(comb, full) < 1e-6  # exact distance tiles: only the fp32 tile-sum grouping differs


def test_c3_naive_knn_deann(c3):
    W, ds, od = c3
    h = MAN["c3"]["h"]
    kern = g.KernelSpec("gaussian", h)
    sel = np.random.default_rng(1).choice(10_000, 12, replace=False)
    Q = W.Q[sel]
    assert _rel(g.naive_kde(ds, kern, Q).values, O.naive_kde(od, "gaussian", h, Q)) < KDE_RTOL
    vals, nbr, smp = g.deann_arrays(ds, kern, Q, 100, 1000, seed=77, query_base=int(sel[0]),
                                    export_neighbors=True, export_samples=True)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], 100)
        np.testing.assert_array_equal(nbr[j], ri)
        ref = O.deann(od, "gaussian", h, NeighborReplay(ri, rd), Q[j], 100, 1000,
                      rng=IndexReplay(77, int(sel[0]) + j, od.n))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-11)


def test_c3_full_batch_deann_statistics(c3):
    W, ds, od = c3
    h = MAN["c3"]["h"]
    kern = g.KernelSpec("gaussian", h)
    exact = g.naive_kde(ds, kern, W.Q).values
    est, _, _ = g.deann_arrays(ds, kern, W.Q, 100, 1000, seed=3)
    sig = (est - exact) / exact
    # DEANN is unbiased (Corollary 1): the mean signed relative error over the 10k
    # independent query streams is 0 within 4 standard errors
    se = sig.std(ddof=1) / np.sqrt(len(sig))
    assert abs(sig.mean()) < 4 * se
    assert np.all(est >= 0)


def test_c4_exponential_and_laplacian():
    W = workloads.make("c4")
    ds, od = g.Dataset.from_array(W.X), O.Data(W.X)
    sel = np.random.default_rng(2).choice(10_000, 8, replace=False)
    Q = W.Q[sel]
    for fam, key in [("exponential", "c4"), ("laplacian", "c4-laplacian")]:
        h = MAN[key]["h"]
        got = g.naive_kde(ds, g.KernelSpec(fam, h), Q).values
        assert _rel(got, O.naive_kde(od, fam, h, Q)) < KDE_RTOL, fam
    h = MAN["c4-laplacian"]["h"]
    vals, nbr, _ = g.deann_arrays(ds, g.KernelSpec("laplacian", h), Q[:4], 50, 500, seed=9, export_neighbors=True)
    for j in range(4):
        ri, rd = O.brute_force_knn(od, Q[j], 50)
        np.testing.assert_array_equal(nbr[j], ri)
        ref = O.deann(od, "laplacian", h, NeighborReplay(ri, rd), Q[j], 50, 500, rng=IndexReplay(9, j, od.n))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-11)


def test_c1_reference_config_end_to_end():
    W = workloads.make("c1")
    ds, od = g.Dataset.from_array(W.X), O.Data(W.X)
    kern = g.KernelSpec("gaussian", 2.0)
    assert _rel(g.naive_kde(ds, kern, W.Q).values, O.naive_kde(od, "gaussian", 2.0, W.Q)) < KDE_RTOL
    vals, nbr, _ = g.deann_arrays(ds, kern, W.Q, 50, 500, seed=11, export_neighbors=True)
    for j in range(0, 1000, 50):
        ri, rd = O.brute_force_knn(od, W.Q[j], 50)
        np.testing.assert_array_equal(nbr[j], ri)
        ref = O.deann(od, "gaussian", 2.0, NeighborReplay(ri, rd), W.Q[j], 50, 500, rng=IndexReplay(11, j, od.n))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-11)


@pytest.mark.slow
def test_c5_scale_out_properties():
    W = workloads.make("c5", nq=4096)
    h = MAN["c5"]["h"]
    kern = g.KernelSpec("gaussian", h)
    ds = g.Dataset.from_array(W.X)
    full = g.naive_kde(ds, kern, W.Q).values
    assert np.all(full > 0)
    # dataset-sharded composition over 4 row shards (what the 4-GPU run computes)
    n = W.X.shape[0]
    acc = np.zeros_like(full)
    for r in range(4):
        lo, hi = (r * n) // 4, ((r + 1) * n) // 4
        acc += g.naive_kde(g.Dataset.from_array(W.X[lo:hi]), kern, W.Q).values * (hi - lo)
    assert _rel(acc / n, full) < 1e-5
    # exact KDE over ALL 8M rows against the fp64 oracle on 16 seeded queries of the batch
    # (the oracle's fp64 copy of the rows is 6 GB of host memory; ~1 s per query)
    od = O.Data(W.X)
    sel16 = np.random.default_rng(5).choice(len(W.Q), 16, replace=False)
    assert _rel(full[sel16], O.naive_kde(od, "gaussian", h, W.Q[sel16])) < KDE_RTOL
    # DEANN at the config's own k = 100, m = 2000 over all 8M rows: neighbour sets equal the
    # oracle's brute force, estimates equal the reference algorithm replaying the GPU's
    # Philox stream
    sel = [0, 1, 2049]
    vals, nbr, _ = g.deann_arrays(ds, kern, W.Q[sel], 100, 2000, seed=5, export_neighbors=True)
    for j, qj in enumerate(sel):
        ri, rd = O.brute_force_knn(od, W.Q[qj], 100)
        np.testing.assert_array_equal(nbr[j], ri)
        ref = O.deann(od, "gaussian", h, NeighborReplay(ri, rd), W.Q[qj], 100, 2000,
                      rng=IndexReplay(5, j, od.n))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-11)


def test_c4_exponential_deann_config_size():
    """c4 DEANN with the exponential kernel at the config's k = 50, m = 500 (tensor-core k-NN on
    784-wide rows + Philox residual), replayed through the reference algorithm."""
    W = workloads.make("c4")
    ds, od = g.Dataset.from_array(W.X), O.Data(W.X)
    h = MAN["c4"]["h"]
    sel = np.random.default_rng(12).choice(10_000, 6, replace=False)
    Q = W.Q[sel]
    vals, nbr, smp = g.deann_arrays(ds, g.KernelSpec("exponential", h), Q, 50, 500, seed=13, query_base=100,
                                    export_neighbors=True, export_samples=True)
    for j in range(len(Q)):
        ri, rd = O.brute_force_knn(od, Q[j], 50)
        np.testing.assert_array_equal(nbr[j], ri)
        assert not np.isin(smp[j], ri).any()  # residual samples exclude the neighbours
        ref = O.deann(od, "exponential", h, NeighborReplay(ri, rd), Q[j], 50, 500,
                      rng=IndexReplay(13, 100 + j, od.n))[0]
        assert vals[j] == pytest.approx(ref, rel=1e-11)


def test_c1_rs_config_m500():
    """c1 RS with m = 500 over the whole 1,000-query batch: the GPU's values equal the reference's
    rs_kde fed the same Philox stream (estimators.py:152-164), through both the batch path and
    the per-query drop-in rs_kde."""
    W = workloads.make("c1")
    ds, od = g.Dataset.from_array(W.X), O.Data(W.X)
    kern = g.KernelSpec("gaussian", 2.0)
    vals, _, smp = g.deann_arrays(ds, kern, W.Q, 0, 500, seed=21, export_samples=True)
    for j in range(0, 1000, 37):
        ref = O.rs_kde(od, "gaussian", 2.0, W.Q[j], 500, IndexReplay(21, j, od.n))
        assert vals[j] == pytest.approx(ref, rel=1e-12)
        np.testing.assert_array_equal(smp[j], IndexReplay(21, j, od.n).integers(0, od.n, size=500))
    sampler = g.PhiloxSampler(21)
    for j in range(5):
        e = g.rs_kde(ds, kern, W.Q[j], 500, sampler)
        assert e.value == pytest.approx(vals[j], rel=1e-14) and e.kernel_evals == 500 and e.samples_used == 500
