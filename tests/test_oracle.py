"""CPU: the NumPy oracle is pinned to the reference's golden vectors.

tests/golden/reference_golden.npz was produced by importing the reference
package itself (tests/golden/make_golden.py).  If these pass, the oracle is a
faithful restatement of the reference on every pinned input, which is what
makes it a valid checker for the GPU path.
"""

import math

import numpy as np
import pytest

from oracle import deann_oracle as O
from oracle.philox import IndexReplay, NeighborReplay, draws, philox4x32_10
from dk_testutil import FAMILIES


def test_kernel_known_answers(golden):
    kat = golden["kat_values"]
    assert kat[0] == 1.0
    assert kat[1] == pytest.approx(math.exp(-1.0), rel=1e-15)
    assert kat[2] == pytest.approx(math.exp(-6.0), rel=1e-12)
    assert kat[3] == pytest.approx(math.exp(-5.0), rel=1e-15)
    assert kat[4] == pytest.approx(math.exp(-1.5), rel=1e-15)
    assert O.kernel_from_distance("gaussian", 1.0, 0.0) == kat[0]
    assert O.kernel_from_distance("exponential", 2.0, 2.0) == kat[1]
    assert O.kernel_from_distance("gaussian", 0.5, 3.0) == kat[2]
    assert O.kernel_pair("exponential", 1.0, [0.0, 0.0], [3.0, 4.0]) == kat[3]
    assert O.kernel_pair("laplacian", 2.0, [1.0, 1.0], [2.0, 3.0]) == kat[4]


def test_kernel_validation():
    with pytest.raises(ValueError):
        O.kernel_from_distance("gaussian", 1.0, -1.0)
    with pytest.raises(ValueError):
        O.kernel_from_distance("gaussian", 1.0, float("nan"))


def test_naive_matches_reference(golden):
    for i in golden["naive_cases"]:
        X, Q, v = golden[f"naive_{i}_X"], golden[f"naive_{i}_Q"], golden[f"naive_{i}_v"]
        h, fi = golden[f"naive_{i}_meta"]
        got = O.naive_kde(O.Data(X), FAMILIES[int(fi)], float(h), Q)
        np.testing.assert_allclose(got, v, rtol=1e-12)


def test_acceptance1_instances(golden):
    for i in range(20):
        X, q = golden[f"acc1_{i}_X"], golden[f"acc1_{i}_q"]
        v, h, fi = golden[f"acc1_{i}_v"]
        got = O.naive_kde(O.Data(X), FAMILIES[int(fi)], float(h), q.reshape(1, -1))[0]
        assert got == pytest.approx(v, rel=1e-12)


def test_knn_matches_reference(golden):
    d = O.Data(golden["knn_X"])
    for j, q in enumerate(golden["knn_Q"]):
        idx, d2 = O.brute_force_knn(d, q, 25)
        np.testing.assert_array_equal(idx, golden["knn_idx"][j])
        np.testing.assert_allclose(d2, golden["knn_d2"][j], rtol=1e-12, atol=1e-12)


def test_sampling_replay_matches_reference(golden):
    d = O.Data(golden["samp_X"])
    seed = int(golden["samp_seed"][0])
    it_rs, it_de = iter(golden["samp_rs"]), iter(golden["samp_deann"])
    for j, q in enumerate(golden["samp_Q"]):
        for fam, h in [("gaussian", 1.3), ("exponential", 1.1), ("laplacian", 2.5)]:
            rs = O.rs_kde(d, fam, h, q, 37, IndexReplay(seed, j, d.n))
            assert rs == pytest.approx(next(it_rs), rel=1e-13)
            val = O.deann(d, fam, h, lambda y, k: O.brute_force_knn(d, y, k), q, 15, 50,
                          rng=IndexReplay(seed + 1, j, d.n))[0]
            assert val == pytest.approx(next(it_de), rel=1e-13)


def test_deann_limits(golden):
    d = O.Data(golden["lim_X"])
    q = golden["lim_q"]
    assert O.naive_kde(d, "gaussian", 1.4, q.reshape(1, -1))[0] == pytest.approx(golden["lim_naive"][0], rel=1e-14)
    v = O.deann(d, "gaussian", 1.4, lambda y, k: O.brute_force_knn(d, y, k), q, 80, 0)[0]
    assert v == pytest.approx(golden["lim_kn"][0], rel=1e-14)
    assert v == pytest.approx(golden["lim_naive"][0], rel=1e-12)


def test_philox_known_answers():
    # Random123 kat_vectors for philox4x32-10
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, exp in kat:
        got = philox4x32_10(np.array([ctr], dtype=np.uint64), key)[0]
        assert [int(v) for v in got] == list(exp)


def test_philox_stream_golden(golden):
    seed = int(golden["samp_seed"][0])
    np.testing.assert_array_equal(draws(seed, 0, 0, 64, 400), golden["philox_q0"])
    np.testing.assert_array_equal(draws(seed, 5, 0, 64, 1_200_000), golden["philox_q5_big"])
    r = IndexReplay(seed, 0, 400)
    a = r.integers(0, 400, 10)
    b = r.integers(0, 400, 54)
    np.testing.assert_array_equal(np.concatenate([a, b]), golden["philox_q0"])


def test_philox_uniformity():
    x = draws(7, 3, 0, 200_000, 1000)
    assert x.min() >= 0 and x.max() < 1000
    counts = np.bincount(x, minlength=1000)
    chi2 = float(((counts - 200.0) ** 2 / 200.0).sum())
    assert chi2 < 1000 + 6 * math.sqrt(2000)  # dof 999


def test_first_m_accepted_semantics():
    # the reference keeps the first `need` non-excluded draws of each batch (estimators.py:225-228)
    d = O.Data(np.random.default_rng(0).normal(size=(60, 3)).astype(np.float32))
    excl_idx = np.arange(0, 60, 3)
    exclude = np.zeros(60, dtype=bool)
    exclude[excl_idx] = True
    stream = draws(5, 0, 0, 5000, 60)
    accepted = stream[~exclude[stream]][:40]
    y = np.zeros(3)
    want = float(O.kernel_rows(d.x64, d.sq_norms, "gaussian", 1.0, accepted, y).sum() / 40)
    got, used = O.rs_excluding(d, "gaussian", 1.0, y, 40, IndexReplay(5, 0, 60), exclude, len(excl_idx))
    assert used == 40
    assert got == pytest.approx(want, rel=1e-14)


def test_neighbor_replay():
    nr = NeighborReplay([3, 1, 2], [0.1, 0.2, 0.3])
    i, d2 = nr(None, 2)
    assert list(i) == [3, 1] and list(d2) == [0.1, 0.2]


def _rsp_setup(golden):
    d = O.Data(golden["rsp_X"])
    return d, golden["rsp_Q"]


def test_rsp_permutation_matches_reference(golden):
    d, _ = _rsp_setup(golden)
    np.testing.assert_array_equal(O.Permuted(d, 80).perm, golden["rsp_perm80"])


def test_rsp_kde_sequences_match_reference(golden):
    d, Q = _rsp_setup(golden)
    it_v, it_c = iter(golden["rsp_vals"]), iter(golden["rsp_cursor"])
    for fi, (fam, h) in enumerate([("gaussian", 1.1), ("exponential", 0.8), ("laplacian", 2.3)]):
        st = O.Permuted(d, 60 + fi, cursor=37 * fi)
        for j, q in enumerate(Q):
            v = O.rsp_kde(st, fam, h, q, [17, 100, 299, 1, 64][j])
            assert v == pytest.approx(next(it_v), rel=1e-12)
            assert st.cursor == next(it_c)


def test_deannp_matches_reference(golden):
    d, Q = _rsp_setup(golden)
    it_v, it_c, it_u = iter(golden["dp_vals"]), iter(golden["dp_cursor"]), iter(golden["dp_used"])
    nb = lambda y, k: O.brute_force_knn(d, y, k)  # noqa: E731
    for fi, (fam, h) in enumerate([("gaussian", 1.1), ("exponential", 0.8), ("laplacian", 2.3)]):
        st = O.Permuted(d, 70 + fi, cursor=290)
        for j, q in enumerate(Q):
            v, _, _, used, trunc, clamped = O.deann_rsp(d, fam, h, nb, q, [10, 0, 25, 299, 5][j],
                                                        [40, 30, 280, 1, 0][j], st)
            assert v == pytest.approx(next(it_v), rel=1e-12)
            assert st.cursor == next(it_c)
            assert [used, int(clamped), int(trunc)] == list(next(it_u))


def test_deannp_batch_cursor_threading(golden):
    d, Q = _rsp_setup(golden)
    nb = lambda y, k: O.brute_force_knn(d, y, k)  # noqa: E731
    st = O.Permuted(d, 80, cursor=123)
    vals = [O.deann_rsp(d, "gaussian", 1.1, nb, q, 12, 50, st)[0] for q in Q]
    np.testing.assert_allclose(vals, golden["dp_batch"], rtol=1e-12)
    assert st.cursor == golden["dp_batch_cursor"][0]
    indep = []
    for j, q in enumerate(Q):
        s2 = O.Permuted(d, 80, cursor=(j * d.n) // len(Q))
        indep.append(O.deann_rsp(d, "gaussian", 1.1, nb, q, 12, 50, s2)[0])
    np.testing.assert_allclose(indep, golden["dp_indep"], rtol=1e-12)


# ------------------------------------------------------------------ inverted file (row f3)


def _ivf_lists(golden, tag):
    rows, off = golden[f"{tag}_rows"], golden[f"{tag}_off"]
    return [rows[off[c]:off[c + 1]] for c in range(len(off) - 1)]


@pytest.mark.parametrize("tag,n,d,C,seed", [("ivf_a", 500, 6, 12, 3), ("ivf_b", 20_000, 16, 64, 7)])
def test_oracle_ivf_matches_reference_goldens(golden, tag, n, d, C, seed):
    X = np.random.default_rng(seed).normal(size=(n, d)).astype(np.float32)
    Q = np.random.default_rng(seed + 1).normal(size=(8, d))
    data = O.Data(X)
    cent, lists = O.ivf_build(data, C, seed)
    np.testing.assert_array_equal(cent, golden[f"{tag}_cent"])
    for a, b in zip(lists, _ivf_lists(golden, tag)):
        np.testing.assert_array_equal(a, b)
    i = 0
    for p in golden[f"{tag}_probes"]:
        for q in Q:
            for formula, key in ((0, "q"), (1, "ann")):
                idx, d2 = O.ivf_query(data, cent, lists, q, 10, int(p), formula)
                gi, gd = golden[f"{tag}_{key}_idx"][i], golden[f"{tag}_{key}_d2"][i]
                np.testing.assert_array_equal(idx, gi[gi >= 0])
                np.testing.assert_allclose(d2, gd[gi >= 0], rtol=1e-12 if formula else 0)
            i += 1


def test_ivf_ann_index_fp32_ranking_pinned(golden):
    """The oracle's IvfAnnIndex restatement (fp32 ranking by (key, probe position), fp64
    re-evaluation; ann.py:276-316) equals the reference on engineered fp32 near-ties, where an
    exact (fp64) ranking of the same probed rows picks different neighbours."""
    differs = 0
    for tag in ("ivf_t1", "ivf_t2"):
        X, Q = golden[f"{tag}_X"], golden[f"{tag}_Q"]
        od = O.Data(X)
        cent, rows, off = golden[f"{tag}_cent"], golden[f"{tag}_rows"], golden[f"{tag}_off"]
        lists = [rows[off[c]:off[c + 1]] for c in range(len(cent))]
        i = 0
        for p in golden[f"{tag}_probes"]:
            for q in Q:
                ri, rd = O.ivf_ann_query(od, cent, lists, q, 10, int(p))
                np.testing.assert_array_equal(ri, golden[f"{tag}_ann_idx"][i][:len(ri)])
                np.testing.assert_array_equal(rd, golden[f"{tag}_ann_d2"][i][:len(rd)])
                fi, _ = O.ivf_query(od, cent, lists, q, 10, int(p), formula=1)
                differs += not np.array_equal(fi, ri)
                i += 1
    assert differs > 0  # the cases do exercise the fp32 tie order
