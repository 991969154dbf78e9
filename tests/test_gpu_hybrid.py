"""Two-precision exact gaussian KDE (capi.cu kde_hybrid, hybrid.cu, tile modes KDE_COLD / KDE_HOT).

The single-pass fp16 sweep sums the tile halves whose kernel sum is small and marks the rest; a
split3 sweep over the listed (query block, tile) pairs sums exactly the marked halves; a per-query
a-posteriori bound on the fp16 part decides which queries are recomputed in split3.  These tests
check the result against the fp64 oracle (naive_kde, estimators.py:144-149) and the split3 path,
the bound itself on pure-fp16 sums, both threshold extremes, forced fallbacks, host queries in
two chunks, and that a bandwidth making most pairs hot turns the path off.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from paper_2107_02736_b200 import _lib  # noqa: E402

H = 0.22392038584059912  # c3's median-1e-3 bandwidth (same generator, fewer rows)
NQ = 4096


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.abs(b)))


def _stats(ds):
    lib = _lib.load()
    v = [ctypes.c_int64() for _ in range(4)]
    _lib.check(lib.dk_kde_stats(ds.handle, *[ctypes.byref(x) for x in v]))
    return [x.value for x in v]


@pytest.fixture(scope="module")
def data():
    X = workloads._c3_rows(3, 200_000)  # 782 tiles: clustered, L2-normalised (config 3's generator)
    Q = workloads._c3_rows(4, NQ).astype(np.float64)
    return X, Q, g.Dataset.from_array(X), O.Data(X)


def _naive_dev(ds, Q, h=H):
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    out = torch.empty(Q.shape[0], dtype=torch.float64, device="cuda")
    g.naive_kde_into(ds, g.KernelSpec("gaussian", h), Qd, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _split3(ds, Q, monkeypatch, h=H):
    monkeypatch.setenv("DK_KDE_HYBRID", "0")
    v = _naive_dev(ds, Q, h)
    monkeypatch.delenv("DK_KDE_HYBRID")
    return v


def test_hybrid_matches_oracle_and_split3(data, monkeypatch):
    X, Q, ds, od = data
    q0, f0, _, _ = _stats(ds)
    got = _naive_dev(ds, Q)
    q1, f1, hot, tot = _stats(ds)
    assert q1 - q0 == NQ and f1 == f0, "the two-precision path served every query without fallbacks"
    assert 0 < hot < 0.25 * tot, (hot, tot)
    sel = np.random.default_rng(1).choice(NQ, 24, replace=False)
    assert _rel(got[sel], O.naive_kde(od, "gaussian", H, Q[sel])) < 1e-5
    assert _rel(got, _split3(ds, Q, monkeypatch)) < 5e-6


def test_fp16_bound_holds_on_pure_fp16_sums(data, monkeypatch):
    """Nothing hot, no fallback: the values are pure fp16 sums, and each stays within the proven
    per-query bound S_cold * expm1(eps_q / 2h^2) of the exact value."""
    X, Q, ds, od = data
    monkeypatch.setenv("DK_HYB_THR", "1e30")
    monkeypatch.setenv("DK_HYB_TOL", "1e30")
    sel = np.random.default_rng(2).choice(NQ, 2048, replace=False)
    Qs = Q[np.sort(sel)]
    fp16 = _naive_dev(ds, Qs)
    exact = O.naive_kde(od, "gaussian", H, Qs[:48])
    mu = X.astype(np.float64).mean(axis=0)
    xn_max = float(np.max(np.sum((X.astype(np.float64) - mu) ** 2, axis=1)))
    Kp = -(-X.shape[1] // 64) * 64
    eps_rel = 1.01 * (2.002 * 2.0 ** -11 + (Kp + 4) * 2.0 ** -24)
    qn = np.sum((Qs[:48] - mu) ** 2, axis=1)
    bound = fp16[:48] * np.expm1(eps_rel * (qn + xn_max) * 1.05 / (2 * H * H))
    err = np.abs(fp16[:48] - exact)
    assert np.all(err <= bound), float(np.max(err / bound))
    assert _rel(fp16[:48], exact) > 1e-6  # really the single-pass values (not split3)


def test_threshold_extremes_and_forced_fallback(data, monkeypatch):
    X, Q, ds, od = data
    Qs = Q[:2048]
    ref = _split3(ds, Qs, monkeypatch)
    monkeypatch.setenv("DK_KDE_HYBRID", "1")  # forced: an all-hot call would turn the path off
    # every half hot: the split3 pass sums everything, the fp16 part is empty (bound 0)
    monkeypatch.setenv("DK_HYB_THR", "-1")
    q0, f0, _, _ = _stats(ds)
    v = _naive_dev(ds, Qs)
    q1, f1, hot, tot = _stats(ds)
    assert f1 == f0 and hot == tot
    assert _rel(v, ref) < 1e-6
    # nothing hot: the bound fails for every query, all recomputed by the split3 fallback
    monkeypatch.setenv("DK_HYB_THR", "1e30")
    v = _naive_dev(ds, Qs)
    _, f2, hot, _ = _stats(ds)
    assert hot == 0 and f2 - f1 == Qs.shape[0]
    assert _rel(v, ref) < 1e-6
    # default threshold, zero tolerance: every query with a fp16 part falls back
    monkeypatch.delenv("DK_HYB_THR")
    monkeypatch.setenv("DK_HYB_TOL", "0")
    v = _naive_dev(ds, Qs)
    _, f3, _, _ = _stats(ds)
    assert f3 - f2 == Qs.shape[0]
    assert _rel(v, ref) < 1e-6


def test_host_queries_two_chunks_and_ragged_batch(data, monkeypatch):
    X, Q, ds, od = data
    Qr = Q[: NQ - 37]  # ragged: not a multiple of 128 or 256
    dev = _naive_dev(ds, Qr)
    host = g.naive_kde(ds, g.KernelSpec("gaussian", H), Qr).values  # pinned host path, two chunks
    assert _rel(dev, host) < 1e-12  # same values; the fp64 partial sums group tiles per batch shape
    sel = np.random.default_rng(3).choice(Qr.shape[0], 8, replace=False)
    assert _rel(host[sel], O.naive_kde(od, "gaussian", H, Qr[sel])) < 1e-5


def test_few_fallbacks_outlier_queries(data, monkeypatch):
    """Queries far from every row (random unit directions) have no hot tile half: their value is
    all fp16 and its bound fails, so they alone are recomputed in split3 (a fallback sweep of a
    single 128-query block, whose partial-sum plan is the widest)."""
    X, Q, ds, od = data
    rng = np.random.default_rng(11)
    out = rng.standard_normal((5, X.shape[1]))
    out /= np.linalg.norm(out, axis=1, keepdims=True)
    Qm = np.concatenate([Q[:2043], out])[rng.permutation(2048)]
    ref = _split3(ds, Qm, monkeypatch)
    q0, f0, _, _ = _stats(ds)
    v = _naive_dev(ds, Qm)
    q1, f1, _, _ = _stats(ds)
    assert q1 - q0 == 2048 and 5 <= f1 - f0 < 128, f1 - f0
    assert _rel(v, ref) < 1e-6


def test_wide_bandwidth_turns_the_path_off(data, monkeypatch):
    """h = 1 on unit vectors: every (block, tile) pair is hot.  Still correct; after one such call
    the handle stops using the two-precision path (it would cost 1 + 3 MMA passes)."""
    X, Q, ds, od = data
    Qs = Q[:2048]
    ref = _split3(ds, Qs, monkeypatch, h=1.0)
    for _ in range(4):
        v = _naive_dev(ds, Qs, h=1.0)
        assert _rel(v, ref) < 1e-6
    q0, _, _, _ = _stats(ds)
    _naive_dev(ds, Qs, h=1.0)
    q1, _, hot, tot = _stats(ds)
    assert q1 == q0 and hot > 0.25 * tot
    sel = np.arange(4)
    assert _rel(v[sel], O.naive_kde(od, "gaussian", 1.0, Qs[sel])) < 1e-5


def test_wide_bandwidth_switches_within_a_multi_batch_call(monkeypatch):
    """A call of several batches reads the first batch's hot fraction at once: with a wide kernel
    the remaining batches take the split3 sweep in the same call (values unchanged)."""
    X = workloads._c3_rows(7, 150_000)
    Q = workloads._c3_rows(8, 3 * 1024).astype(np.float64)
    ds = g.Dataset.from_array(X)
    ref = _split3(ds, Q, monkeypatch, h=1.0)
    monkeypatch.setenv("DK_HYB_BATCH", "1024")
    q0, _, _, _ = _stats(ds)
    v = _naive_dev(ds, Q, h=1.0)
    q1, _, hot, tot = _stats(ds)
    assert hot > 0.25 * tot and q1 - q0 == 1024  # the first batch only
    assert _rel(v, ref) < 1e-6


def test_handles_release_the_two_precision_operands():
    """Fit -> two-precision KDE (ball-sorted rows, fp16 and split3 operands, workspace) -> free,
    three times: the device memory comes back (no per-handle leak of the new operands)."""
    X = workloads._c3_rows(21, 140_000)
    Q = workloads._c3_rows(22, 2048).astype(np.float64)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(3):
        ds = g.Dataset.from_array(X)
        g.naive_kde(ds, g.KernelSpec("gaussian", H), Q)
        assert _stats(ds)[0] == Q.shape[0]
        ds.free()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20, (free0, free1)


def test_far_queries_on_the_two_precision_path():
    """A batch large enough for the two-precision path with queries far from every row: their values lie
    under the fp32 epilogue's range and are recomputed in fp64 (redo.cu), as on the split3 path."""
    rng = np.random.default_rng(3)
    n, d = 140_000, 16
    centers = rng.normal(scale=3.0, size=(40, d))
    X = (centers[rng.integers(0, 40, n)] + 0.3 * rng.normal(size=(n, d))).astype(np.float32)
    Q = centers[rng.integers(0, 40, 2304)] + 0.3 * rng.normal(size=(2304, d))
    Q[:16] += 25.0
    h = 0.9
    ds = g.Dataset.from_array(X)
    got = g.naive_kde(ds, g.KernelSpec("gaussian", h), Q).values
    c = ctypes.c_int64(-1)
    _lib.check(_lib.load().dk_kde_redo_count(ds.handle, ctypes.byref(c)))
    sel = np.r_[0:16, 16:2304:97]
    ref = O.naive_kde(O.Data(X), "gaussian", h, Q[sel])
    assert ref[:16].max() < 1e-40 and c.value >= 16
    np.testing.assert_allclose(got[sel][:16], ref[:16], rtol=1e-9)
    live = ref[16:] > 1e-30
    np.testing.assert_allclose(got[sel][16:][live], ref[16:][live], rtol=1e-5)
