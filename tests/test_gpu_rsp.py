"""GPU permuted sampler (RSP / DEANNP) against the reference goldens and the oracle.

The permuted sampler is deterministic (numpy PCG64 permutation, cursor
arithmetic), so the GPU must reproduce the reference's values and cursors
exactly — values to 1e-12 (fp64 direct differences vs the reference's fp64
matvec), cursors and sample counts bit-for-bit.
"""

import numpy as np
import pytest

import paper_2107_02736_b200 as g
from oracle import deann_oracle as O

pytestmark = pytest.mark.gpu

FAMS = [("gaussian", 1.1), ("exponential", 0.8), ("laplacian", 2.3)]


def test_rsp_kde_sequences_match_reference(golden):
    ds = g.Dataset.from_array(golden["rsp_X"])
    Q = golden["rsp_Q"]
    it_v, it_c = iter(golden["rsp_vals"]), iter(golden["rsp_cursor"])
    for fi, (fam, h) in enumerate(FAMS):
        st = g.RspState.from_dataset(ds, 60 + fi, cursor=37 * fi)
        for j, q in enumerate(Q):
            m = [17, 100, 299, 1, 64][j]
            est = g.rsp_kde(st, g.KernelSpec(fam, h), q, m)
            assert est.value == pytest.approx(next(it_v), rel=1e-12)
            assert st.cursor == next(it_c)
            assert est.samples_used == est.kernel_evals == m


def test_deannp_matches_reference(golden):
    ds = g.Dataset.from_array(golden["rsp_X"])
    Q = golden["rsp_Q"]
    bf = g.BruteForceIndex(ds)
    it_v, it_c, it_u = iter(golden["dp_vals"]), iter(golden["dp_cursor"]), iter(golden["dp_used"])
    for fi, (fam, h) in enumerate(FAMS):
        st = g.RspState.from_dataset(ds, 70 + fi, cursor=290)
        for j, q in enumerate(Q):
            e = g.deann(ds, g.KernelSpec(fam, h), bf, q, [10, 0, 25, 299, 5][j], [40, 30, 280, 1, 0][j],
                        rsp_state=st)
            assert e.value == pytest.approx(next(it_v), rel=1e-12)
            assert st.cursor == next(it_c)
            assert [e.samples_used, int(e.clamped), int(e.truncated)] == list(next(it_u))
            assert e.kernel_evals == e.neighbors_used + e.samples_used


def test_deannp_batch_shared_and_independent(golden):
    ds = g.Dataset.from_array(golden["rsp_X"])
    Q = golden["rsp_Q"]
    shared = g.RspState.from_dataset(ds, 80, cursor=123)
    np.testing.assert_array_equal(shared.permuted.permutation, golden["rsp_perm80"])
    bf = g.BruteForceIndex(ds)
    batch = g.deann_batch(ds, g.KernelSpec("gaussian", 1.1), bf, Q, 12, 50, rsp_state=shared)
    np.testing.assert_allclose([e.value for e in batch], golden["dp_batch"], rtol=1e-12)
    assert shared.cursor == golden["dp_batch_cursor"][0]
    cur = shared.cursor
    indep = g.deann_batch(ds, g.KernelSpec("gaussian", 1.1), bf, Q, 12, 50, rsp_state=shared,
                          independent_cursors=True)
    np.testing.assert_allclose([e.value for e in indep], golden["dp_indep"], rtol=1e-12)
    assert shared.cursor == cur  # independent cursors leave the shared state alone


@pytest.mark.parametrize("family,h", FAMS)
def test_deannp_large_batch_vs_oracle(family, h):
    rng = np.random.default_rng(9)
    X = rng.normal(size=(40_000, 24)).astype(np.float32)
    Q = rng.normal(size=(48, 24))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    st = g.RspState.from_dataset(ds, 5, cursor=39_000)   # walks wrap around the end
    got = g.deann_batch(ds, g.KernelSpec(family, h), g.BruteForceIndex(ds), Q, 40, 700, rsp_state=st)
    ost = O.Permuted(od, 5, cursor=39_000)
    nb = lambda y, k: O.brute_force_knn(od, y, k)  # noqa: E731
    for j, q in enumerate(Q):
        ref = O.deann_rsp(od, family, h, nb, q, 40, 700, ost)
        assert got[j].value == pytest.approx(ref[0], rel=1e-12)
    assert st.cursor == ost.cursor


def test_rsp_cycling_touches_every_row_once():
    # acceptance 11 (test_acceptance.py:397-419)
    n = 512
    rng = np.random.default_rng(111)
    X = rng.normal(size=(n, 5)).astype(np.float32)
    kernel = g.KernelSpec("exponential", 1.5)
    q = rng.normal(size=5)
    ds = g.Dataset.from_array(X)
    st = g.RspState.from_dataset(ds, 3)
    weighted = sum(g.rsp_kde(st, kernel, q, m).value * m for m in [97, 101, 128, 150, 36])
    exact_total = O.naive_kde(O.Data(X), "exponential", 1.5, q.reshape(1, -1))[0] * n
    assert abs(weighted - exact_total) / exact_total <= 1e-12
    assert st.cursor == 0


def test_rsp_validation_and_reference_objects():
    X = np.random.default_rng(1).normal(size=(30, 3)).astype(np.float32)
    ds = g.Dataset.from_array(X)
    st = g.RspState.from_dataset(ds, 0)
    with pytest.raises(ValueError):
        g.rsp_kde(st, g.KernelSpec("gaussian", 1.0), np.zeros(3), 0)
    with pytest.raises(ValueError):
        g.rsp_kde(st, g.KernelSpec("gaussian", 1.0), np.zeros(3), 31)
    other = g.RspState.from_dataset(g.Dataset.from_array(X[:29]), 0)
    with pytest.raises(ValueError):
        g.deann(ds, g.KernelSpec("gaussian", 1.0), g.BruteForceIndex(ds), np.zeros(3), 2, 5, rsp_state=other)

    class RefPermuted:  # duck-typed reference PermutedDataset / RspState
        def __init__(self, perm):
            class B:
                pass
            self.base = B()
            self.base.data = X[perm]
            self.permutation = perm
            self.inverse_permutation = np.argsort(perm)

        @property
        def n(self):
            return len(self.permutation)

    class RefState:
        def __init__(self, p, cursor):
            self.permuted, self.cursor = p, cursor

        @property
        def n(self):
            return self.permuted.n

    perm = np.random.default_rng(0).permutation(30).astype(np.int64)
    rs = RefState(RefPermuted(perm), 25)
    v = g.rsp_kde(rs, g.KernelSpec("gaussian", 1.0), X[0], 10).value
    ost = O.Permuted(O.Data(X), 0, cursor=25)
    assert v == pytest.approx(O.rsp_kde(ost, "gaussian", 1.0, X[0], 10), rel=1e-12)
    assert rs.cursor == ost.cursor == 5
