"""Operands with norm columns (prep.cu: A = [q | w | -b(q)], B = [x | -b(x) | w], the MMA yields
-d2/2 and the gaussian epilogue multiplies once per pair; tile mode KDE_GAUSS_AUG / KDE_COLD_AUG).

Exact integer rows: the norm split is exact, so d2 is exact and the KDE matches the fp64 oracle
(naive_kde, estimators.py:144-149) to the exponential's own rounding — checked next to the exact-mode
limit (squared norms just under 2^23, the largest b1).  d = 50 / 57 / 100 keep the columns in the
K padding; d = 64 has none, so they go to the 16-column tail operand (one more 16-wide MMA step on
32-byte-swizzled tiles), also for the two-precision sweep's fp16 pass (KDE_COLD_AUG); DK_AUG_TAIL=0
falls back to the plain epilogue.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from paper_2107_02736_b200 import _lib  # noqa: E402


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.mark.parametrize("d", [50, 57, 64, 100])
def test_exact_integer_rows_near_the_norm_limit(d):
    rng = np.random.default_rng(d)
    vmax = int(np.sqrt((2 ** 23 - 1) / d))  # squared norms up to just under 2^23
    X = rng.integers(0, vmax + 1, size=(20_000, d)).astype(np.float32)
    X[:64] = vmax  # rows at the limit: b1 = floor(|x|^2 / 4096) at its largest
    Q = rng.integers(0, vmax + 1, size=(300, d)).astype(np.float64)
    Q[:3] = vmax
    ds = g.Dataset.from_array(X)
    assert ds.exact_mode
    h = 0.35 * vmax * np.sqrt(d)
    got = g.naive_kde(ds, g.KernelSpec("gaussian", h), Q).values
    ref = O.naive_kde(O.Data(X), "gaussian", h, Q)
    assert _rel(got, ref) < 2e-6


def test_two_precision_with_tail_norm_columns(monkeypatch):
    """d = 64: the fp16 pass of the two-precision KDE takes its norm columns from the tail operand."""
    X = workloads._c3_rows(3, 160_000)[:, :64].copy()
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Q = workloads._c3_rows(4, 2048).astype(np.float64)[:, :64].copy()
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    ds = g.Dataset.from_array(X)
    h = 0.2
    got = g.naive_kde(ds, g.KernelSpec("gaussian", h), Q).values
    monkeypatch.setenv("DK_KDE_HYBRID", "0")
    ref3 = g.naive_kde(ds, g.KernelSpec("gaussian", h), Q).values
    assert _rel(got, ref3) < 5e-6
    sel = np.arange(0, 2048, 256)
    assert _rel(got[sel], O.naive_kde(O.Data(X), "gaussian", h, Q[sel])) < 1e-5


def test_exact_tail_matches_plain_epilogue_in_a_fresh_process():
    """The tail path (d = 128, c2's shape) against the plain epilogue of the same library
    (DK_AUG_TAIL=0, read once per process: run in a subprocess) on integer rows: both exact d2,
    so the values agree to the exponentials' rounding."""
    import os
    import subprocess
    import sys

    from dk_testutil import REPO

    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_2107_02736_b200 as g\n"
        "rng = np.random.default_rng(3)\n"
        "X = rng.integers(0, 256, size=(30000, 128)).astype(np.float32)\n"
        "Q = rng.integers(0, 256, size=(5000, 128)).astype(np.float64)\n"
        "ds = g.Dataset.from_array(X)\n"
        "np.save(sys.argv[1], g.naive_kde(ds, g.KernelSpec('gaussian', 900.0), Q).values)\n" % REPO
    )
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        outs = []
        for env_tail in ("1", "0"):
            path = os.path.join(td, f"v{env_tail}.npy")
            env = dict(os.environ, DK_AUG_TAIL=env_tail)
            subprocess.run([sys.executable, "-c", code, path], check=True, env=env)
            outs.append(np.load(path))
    assert _rel(outs[0], outs[1]) < 2e-6


def test_tail_integer_rows_with_fractional_and_host_query_chunks():
    """d = 128 integer rows (the tail path): a host batch of two chunks whose second chunk has a
    fractional query — that chunk's speculative exact sweep skips itself and is redone in split3
    after both chunks are enqueued; the first chunk stays exact."""
    rng = np.random.default_rng(17)
    X = rng.integers(0, 256, size=(20_000, 128)).astype(np.float32)
    Q = rng.integers(0, 256, size=(4096, 128)).astype(np.float64)
    Q[4000] += 0.5
    ds, od = g.Dataset.from_array(X), O.Data(X)
    assert ds.exact_mode
    h = 900.0
    got = g.naive_kde(ds, g.KernelSpec("gaussian", h), Q).values
    sel = np.array([0, 1, 1023, 1024, 2048, 4000, 4095])
    assert _rel(got[sel], O.naive_kde(od, "gaussian", h, Q[sel])) < 2e-6


def test_two_precision_on_dataset_shards(monkeypatch):
    """Dataset-sharded handles (global_offset / global_n, each shard >= 512 tiles) take the
    two-precision path too: their contributions to the global mean add up to the whole dataset's."""
    X = workloads._c3_rows(11, 2 * 140_000)
    Q = workloads._c3_rows(12, 2048).astype(np.float64)
    h = 0.2239
    n = X.shape[0]
    full = g.naive_kde(g.Dataset.from_array(X), g.KernelSpec("gaussian", h), Q).values
    acc = np.zeros_like(full)
    for lo, hi in ((0, n // 2), (n // 2, n)):
        sh = g.Dataset.from_array(X[lo:hi], global_offset=lo, global_n=n)
        acc += g.naive_kde(sh, g.KernelSpec("gaussian", h), Q).values
        lib = _lib.load()
        import ctypes

        v = [ctypes.c_int64() for _ in range(4)]
        _lib.check(lib.dk_kde_stats(sh.handle, *[ctypes.byref(x) for x in v]))
        assert v[0].value == Q.shape[0]  # served two-precision
    assert _rel(acc, full) < 5e-6
    sel = np.arange(0, 2048, 512)
    assert _rel(full[sel], O.naive_kde(O.Data(X), "gaussian", h, Q[sel])) < 1e-5
