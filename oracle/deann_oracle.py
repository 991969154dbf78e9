"""CPU oracle for the DEANN KDE query path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only tests/, the smoke() of
__graft_entry__.py and bench.py's cpu_baseline / --impl reference arm may
import it.  It restates, in plain NumPy (fp64 throughout), the algorithms of
the reference package `deann` 0.1.0 (/root/reference/pkg/src/deann/), each
function citing the lines it follows.  It is pinned against golden vectors
produced by importing the real reference (tests/golden/make_golden.py ->
tests/golden/*.npz, checked by tests/test_oracle.py).

The arithmetic dependency of the reference is NumPy/OpenBLAS (unpinned,
`numpy>=1.24`, pyproject.toml:10): DGEMM in batch_sqdist, einsum norms,
np.exp, argpartition/lexsort, PCG64 Generator.integers.  This restatement
uses the same NumPy calls for the same steps, so agreement with the
reference is at the 1e-15 level.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "row_norms", "batch_sqdist", "kernel_from_distance", "kernel_from_sql2", "kernel_rows", "naive_kde",
    "rs_kde", "rs_excluding", "smallest_k", "brute_force_knn", "deann", "deann_batch", "kernel_pair",
]

BLOCK_ENTRIES = 4_000_000  # estimators.py:54
CLAMP_REL = 1e-3           # distance.py:25


class NormConsistencyError(RuntimeError):
    """distance.py:28-29"""


def as_rows(data) -> np.ndarray:
    """Dataset.from_array storage: C-contiguous float32 (data.py:55)."""
    return np.ascontiguousarray(data, dtype=np.float32)


def row_norms(x32: np.ndarray) -> np.ndarray:
    """fp64 squared row norms via einsum (data.py:63-64)."""
    d64 = x32.astype(np.float64)
    return np.einsum("ij,ij->i", d64, d64)


def kernel_from_distance(family: str, h: float, dist):
    """kernels.py:65-83: validates finite & >= 0, then exp(-d/(2h^2)) or exp(-d/h)."""
    scalar = np.isscalar(dist) or np.ndim(dist) == 0
    d = np.asarray(dist, dtype=np.float64)
    if not np.all(np.isfinite(d)):
        raise ValueError("distance must be finite")
    if np.any(d < 0.0):
        raise ValueError("distance must be nonnegative")
    out = np.exp(-d / (2.0 * h * h)) if family == "gaussian" else np.exp(-d / h)
    return float(out) if scalar else out


def kernel_pair(family: str, h: float, x, y) -> float:
    """kernels.py:86-106: scalar oracle with the family's own metric."""
    diff = np.asarray(x, dtype=np.float64).ravel() - np.asarray(y, dtype=np.float64).ravel()
    if family == "gaussian":
        dist = float(diff @ diff)
    elif family == "exponential":
        dist = math.sqrt(float(diff @ diff))
    else:
        dist = float(np.abs(diff).sum())
    return kernel_from_distance(family, h, dist)


def _clamp(d2: np.ndarray, scale: float) -> np.ndarray:
    """distance.py:58-66"""
    tol = CLAMP_REL * max(scale, 1.0)
    worst = d2.min() if d2.size else 0.0
    if worst < -tol:
        raise NormConsistencyError(f"batch distance {worst:g} below clamp tolerance {-tol:g}")
    np.maximum(d2, 0.0, out=d2)
    return d2


def batch_sqdist(q: np.ndarray, x64: np.ndarray, sq_norms: np.ndarray) -> np.ndarray:
    """distance.py:69-85: ||q||^2 + ||x||^2 - 2 q.x in fp64, clamped."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    q_norms = np.einsum("ij,ij->i", q, q)
    d2 = q @ x64.T
    d2 *= -2.0
    d2 += q_norms[:, None]
    d2 += sq_norms[None, :]
    scale = float(q_norms.max(initial=0.0) + sq_norms.max(initial=0.0))
    return _clamp(d2, scale)


def kernel_from_sql2(family: str, h: float, d2: np.ndarray) -> np.ndarray:
    """estimators.py:99-103"""
    if family == "gaussian":
        return kernel_from_distance(family, h, d2)
    return kernel_from_distance(family, h, np.sqrt(d2))


def kernel_rows(x64: np.ndarray, sq_norms: np.ndarray, family: str, h: float, rows: np.ndarray,
                y: np.ndarray) -> np.ndarray:
    """estimators.py:106-119"""
    if len(rows) == 0:
        return np.empty(0, dtype=np.float64)
    x = x64[rows]
    if family == "laplacian":
        return kernel_from_distance(family, h, np.abs(x - y).sum(axis=1))
    d2 = x @ y
    d2 *= -2.0
    d2 += sq_norms[rows]
    d2 += float(y @ y)
    np.maximum(d2, 0.0, out=d2)
    return kernel_from_sql2(family, h, d2)


class Data:
    """Oracle-side dataset: fp32 rows, fp64 copy, fp64 norms (data.py:45-83)."""

    def __init__(self, data):
        self.x32 = as_rows(data)
        self.x64 = self.x32.astype(np.float64)
        self.sq_norms = row_norms(self.x32)

    @property
    def n(self) -> int:
        return self.x32.shape[0]

    @property
    def d(self) -> int:
        return self.x32.shape[1]


def naive_kde(data: Data, family: str, h: float, queries) -> np.ndarray:
    """estimators.py:122-149 (L2 via blocked batch_sqdist, L1 via per-query row blocks)."""
    q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    if q.shape[1] != data.d:
        raise ValueError(f"dimension mismatch: queries d={q.shape[1]}, dataset d={data.d}")
    n = data.n
    values = np.empty(q.shape[0], dtype=np.float64)
    if family == "laplacian":
        step = max(1, BLOCK_ENTRIES // data.d)
        for j, y in enumerate(q):
            acc = 0.0
            for lo in range(0, n, step):
                dist = np.abs(data.x64[lo: lo + step] - y).sum(axis=1)
                acc += float(kernel_from_distance(family, h, dist).sum())
            values[j] = acc / n
        return values
    block = max(1, BLOCK_ENTRIES // n)
    for lo in range(0, q.shape[0], block):
        hi = min(q.shape[0], lo + block)
        d2 = batch_sqdist(q[lo:hi], data.x64, data.sq_norms)
        values[lo:hi] = kernel_from_sql2(family, h, d2).mean(axis=1)
    return values


def rs_kde(data: Data, family: str, h: float, query, m: int, rng) -> float:
    """estimators.py:152-164 (rng: anything with .integers(low, high, size))."""
    if m < 1:
        raise ValueError(f"m={m} must be >= 1")
    y = np.asarray(query, dtype=np.float64).ravel()
    draws = rng.integers(0, data.n, size=m)
    return float(kernel_rows(data.x64, data.sq_norms, family, h, draws, y).mean())


def rs_excluding(data: Data, family: str, h: float, y: np.ndarray, m: int, rng, exclude, n_excluded: int):
    """estimators.py:203-233: first-m-accepted rejection sampling restricted to X \\ X1."""
    n = data.n
    total = 0.0
    accepted = 0
    while accepted < m:
        need = m - accepted
        if n_excluded == 0:
            batch = need
        else:
            batch = min(math.ceil(need * n / (n - n_excluded)) + 8, max(4 * need, 65536))
        draws = rng.integers(0, n, size=batch)
        if n_excluded:
            draws = draws[~exclude[draws]]
        draws = draws[:need]
        if len(draws) == 0:
            continue
        total += float(kernel_rows(data.x64, data.sq_norms, family, h, draws, y).sum())
        accepted += len(draws)
    return total / m, m


def smallest_k(d2: np.ndarray, ids: np.ndarray, k: int):
    """ann.py:82-102: k smallest, boundary widening, stable argsort, lexsort on ties."""
    k = min(k, len(d2))
    if k < len(d2):
        part = np.argpartition(d2, k - 1)[:k]
        boundary = d2[part].max()
        cand = np.flatnonzero(d2 <= boundary)
        cd = d2[cand]
    else:
        cand = np.arange(len(d2))
        cd = d2
    order = np.argsort(cd, kind="stable")
    if len(order) > 1 and np.any(np.diff(cd[order]) == 0.0):
        order = np.lexsort((ids[cand], cd))
    sel = cand[order[:k]]
    return ids[sel], d2[sel]


def brute_force_knn(data: Data, query, k: int):
    """ann.py:105-111 -> (indices int64, sq_distances fp64)."""
    if not 1 <= k <= data.n:
        raise ValueError(f"k={k} out of range [1, {data.n}]")
    d2 = batch_sqdist(np.asarray(query, dtype=np.float64).reshape(1, -1), data.x64, data.sq_norms)[0]
    return smallest_k(d2, np.arange(data.n, dtype=np.int64), k)


def deann(data: Data, family: str, h: float, neighbors, query, k: int, m: int, rng=None):
    """estimators.py:306-379 with the uniform sampler.

    `neighbors` is a callable (y, k) -> (indices, sq_distances) (the AnnIndex
    black box, e.g. brute_force_knn or a replay of GPU neighbours).
    Returns (value, kernel_evals, k_hat, samples_used, truncated).
    """
    n = data.n
    if not 0 <= k <= n:
        raise ValueError(f"k={k} out of range [0, {n}]")
    if m < 0:
        raise ValueError(f"m={m} must be >= 0")
    if m > 0 and k >= n:
        raise ValueError("m > 0 requires k + 1 <= n so the remainder is nonempty")
    if m > 0 and rng is None:
        raise ValueError("give exactly one of rng= or rsp_state= when m > 0")
    y = np.asarray(query, dtype=np.float64).ravel()
    if y.shape[0] != data.d:
        raise ValueError(f"dimension mismatch: query d={y.shape[0]}, dataset d={data.d}")
    if k > 0:
        idx, sqd = neighbors(y, k)
        x1 = np.asarray(idx, dtype=np.int64)
    else:
        x1, sqd = np.empty(0, dtype=np.int64), None
    k_hat = len(x1)
    if k_hat == 0:
        z1 = 0.0
    elif family == "laplacian":
        z1 = float(kernel_rows(data.x64, data.sq_norms, family, h, x1, y).mean())
    else:
        z1 = float(kernel_from_sql2(family, h, np.asarray(sqd, dtype=np.float64)).mean())
    if m == 0:
        return (k_hat / n) * z1, k_hat, k_hat, 0, k_hat < n
    if k_hat:
        exclude = np.zeros(n, dtype=bool)
        exclude[x1] = True
    else:
        exclude = None
    z2, used = rs_excluding(data, family, h, y, m, rng, exclude, k_hat)
    value = (k_hat / n) * z1 + ((n - k_hat) / n) * z2
    return value, k_hat + used, k_hat, used, False


def deann_batch(data: Data, family: str, h: float, neighbors, queries, k: int, m: int, rng=None):
    """estimators.py:382-410 (uniform sampler): a loop of deann in query order."""
    q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    return [deann(data, family, h, neighbors, q[j], k, m, rng=rng)[0] for j in range(q.shape[0])]


# ---------------------------------------------------------------- permuted sampler (RSP / DEANNP)


class Permuted:
    """PermutedDataset + RspState cursor (data.py:103-117, 214-233; estimators.py:83-96)."""

    def __init__(self, data: "Data", seed: int, cursor: int = 0):
        rng = np.random.default_rng(seed)
        self.perm = rng.permutation(data.n).astype(np.int64)        # data.py:226
        self.inverse = np.empty_like(self.perm)
        self.inverse[self.perm] = np.arange(data.n, dtype=np.int64)  # data.py:227-228
        self.base = Data(data.x32[self.perm])                        # rows move with the permutation
        self.cursor = int(cursor)

    @property
    def n(self) -> int:
        return self.base.n


def window_ranges(n: int, start: int, count: int):
    """distance.py:88-98"""
    if start + count <= n:
        return [(start, start + count)]
    return [(start, n), (0, start + count - n)]


def _block_values(base: Data, family: str, h: float, y: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """estimators.py:236-246 (one matvec per contiguous block)."""
    if family == "laplacian":
        return kernel_from_distance(family, h, np.abs(base.x64[lo:hi] - y).sum(axis=1))
    d2 = base.x64[lo:hi] @ y
    d2 *= -2.0
    d2 += base.sq_norms[lo:hi]
    d2 += float(y @ y)
    np.maximum(d2, 0.0, out=d2)
    return kernel_from_sql2(family, h, d2)


def rsp_kde(state: Permuted, family: str, h: float, query, m: int) -> float:
    """estimators.py:180-200: mean over the next m permuted rows (wrapping); cursor += m."""
    n = state.n
    if not 1 <= m <= n:
        raise ValueError(f"m={m} out of range [1, {n}]")
    y = np.asarray(query, dtype=np.float64).ravel()
    total = sum(float(_block_values(state.base, family, h, y, lo, hi).sum())
                for lo, hi in window_ranges(n, state.cursor, m))
    state.cursor = (state.cursor + m) % n
    return total / m


def rsp_excluding(state: Permuted, family: str, h: float, y, m: int, exclude, n_excluded: int):
    """estimators.py:249-303: walk from the cursor skipping excluded ORIGINAL ids until m
    rows are accepted or a full pass completes; the cursor advances past skipped rows."""
    n = state.n
    if n_excluded == 0:
        count = min(m, n)
        total = sum(float(_block_values(state.base, family, h, y, lo, hi).sum())
                    for lo, hi in window_ranges(n, state.cursor, count))
        state.cursor = (state.cursor + count) % n
        return total / count, count, count < m
    perm = state.perm
    advanced = taken = 0
    total = 0.0
    while taken < m and advanced < n:
        pos = (state.cursor + advanced) % n
        chunk = min(n - advanced, max(m - taken + 64, 64))
        consumed = chunk
        for lo, hi in window_ranges(n, pos, chunk):
            keep = ~exclude[perm[lo:hi]]
            kept = int(np.count_nonzero(keep))
            need = m - taken
            if kept >= need:
                cut = int(np.flatnonzero(keep)[need - 1]) + 1
                keep = keep[:cut]
                hi = lo + cut
                consumed = (lo - pos) % n + cut
                kept = need
            if kept:
                vals = _block_values(state.base, family, h, y, lo, hi)
                total += float(vals[keep].sum())
                taken += kept
            if taken == m:
                break
        advanced += consumed
    state.cursor = (state.cursor + advanced) % n
    if taken == 0:
        return 0.0, 0, True
    return total / taken, taken, taken < m


def deann_rsp(data: Data, family: str, h: float, neighbors, query, k: int, m: int, state: Permuted):
    """estimators.py:306-379 with the permuted sampler.  Returns (value, evals, k_hat, used, truncated, clamped)."""
    n = data.n
    if state.n != n:
        raise ValueError("rsp_state was built for a different dataset size")
    y = np.asarray(query, dtype=np.float64).ravel()
    if k > 0:
        idx, sqd = neighbors(y, k)
        x1 = np.asarray(idx, dtype=np.int64)
    else:
        x1, sqd = np.empty(0, dtype=np.int64), None
    k_hat = len(x1)
    if k_hat == 0:
        z1 = 0.0
    elif family == "laplacian":
        z1 = float(kernel_rows(data.x64, data.sq_norms, family, h, x1, y).mean())
    else:
        z1 = float(kernel_from_sql2(family, h, np.asarray(sqd, dtype=np.float64)).mean())
    if m == 0:
        return (k_hat / n) * z1, k_hat, k_hat, 0, k_hat < n, False
    exclude = np.zeros(n, dtype=bool)
    exclude[x1] = True
    z2, used, clamped = rsp_excluding(state, family, h, y, m, exclude if k_hat else None, k_hat)
    value = (k_hat / n) * z1 + ((n - k_hat) / n) * z2
    return value, k_hat + used, k_hat, used, False, clamped


# ---------------------------------------------------------------- inverted file (row f3)

KMEANS_MAX_ITER = 25   # ann.py:45
KMEANS_REL_TOL = 1e-4  # ann.py:46


def centroid_sqdists(x64: np.ndarray, sq_norms: np.ndarray, cent: np.ndarray) -> np.ndarray:
    """ann.py:142-149: ((x.c) * -2 + |x|^2) + |c|^2, clamped at 0."""
    cn = np.einsum("ij,ij->i", cent, cent)
    out = (x64 @ cent.T) * -2.0
    out += sq_norms[:, None]
    out += cn[None, :]
    return np.maximum(out, 0.0)


def kmeans_pp(x64: np.ndarray, n_clusters: int, rng) -> np.ndarray:
    """ann.py:152-169: D^2 seeding; one rng.choice(p=...) per further centroid."""
    n, d = x64.shape
    cent = np.zeros((n_clusters, d))
    cent[0] = x64[int(rng.integers(n))]
    diff = x64 - cent[0]
    dmin = np.einsum("ij,ij->i", diff, diff)
    for c in range(1, n_clusters):
        mass = dmin.sum()
        row = int(rng.integers(n)) if mass <= 0.0 else int(rng.choice(n, p=dmin / mass))
        cent[c] = x64[row]
        diff = x64 - cent[c]
        dmin = np.minimum(dmin, np.einsum("ij,ij->i", diff, diff))
    return cent


def ivf_build(data: Data, n_clusters: int, seed: int):
    """ann.py:172-199 -> (centroids (C, d), list of member arrays).

    Note the convergence test uses prev = +inf on the first pass, so inf - wcss <=
    tol * inf holds and the reference stops after one Lloyd update; restated as is.
    """
    n = data.n
    if not 1 <= n_clusters <= n:
        raise ValueError(f"n_clusters={n_clusters} out of range [1, {n}]")
    rng = np.random.default_rng(seed)
    cent = kmeans_pp(data.x64, n_clusters, rng)
    prev = math.inf
    for _ in range(KMEANS_MAX_ITER):
        d2 = centroid_sqdists(data.x64, data.sq_norms, cent)
        lab = np.argmin(d2, axis=1)
        wcss = float(d2[np.arange(n), lab].sum())
        for c in range(n_clusters):
            sel = lab == c
            if sel.any():
                cent[c] = data.x64[sel].mean(axis=0)
        if prev - wcss <= KMEANS_REL_TOL * max(prev, 1e-300):
            break
        prev = wcss
    lab = np.argmin(centroid_sqdists(data.x64, data.sq_norms, cent), axis=1)
    return cent, [np.flatnonzero(lab == c).astype(np.int64) for c in range(n_clusters)]


def _probe(cent: np.ndarray, y: np.ndarray, n_probe: int, formula: int) -> np.ndarray:
    """n_probe nearest centroids, ties to the lower id: formula 0 = sum (c - y)^2
    (ivf_query, ann.py:212-214), 1 = (C y) * -2 + |c|^2 (IvfAnnIndex, ann.py:262-275)."""
    if formula == 0:
        diff = cent - y
        cd = np.einsum("ij,ij->i", diff, diff)
    else:
        cd = (cent @ y) * -2.0 + np.einsum("ij,ij->i", cent, cent)
    ids = np.arange(len(cent), dtype=np.int64)
    return ids[np.lexsort((ids, cd))[:n_probe]]


def ivf_query(data: Data, cent: np.ndarray, lists, query, k: int, n_probe: int, formula: int = 0):
    """ann.py:204-230 -> (indices, sq_distances): exact k smallest among the probed lists."""
    y = np.asarray(query, dtype=np.float64).ravel()
    members = [lists[c] for c in _probe(cent, y, n_probe, formula) if len(lists[c])]
    if not members:
        return np.empty(0, np.int64), np.empty(0)
    cand = np.concatenate(members)
    d2 = (data.x64[cand] @ y) * -2.0
    d2 += data.sq_norms[cand]
    d2 += float(y @ y)
    return smallest_k(np.maximum(d2, 0.0), cand, k)


def ivf_ann_query(data: Data, cent: np.ndarray, lists, query, k: int, n_probe: int):
    """IvfAnnIndex.query (ann.py:243-316) restated with the reference's own arithmetic: probe by
    (C y) * -2 + |c|^2 with (distance, id) order; candidate ranking in SINGLE precision over the
    list-contiguous fp32 rows (vectors32 @ y32, then norms32 - 2 * dot, numpy fp32 — the BLAS
    sgemv of the reference), argpartition boundary widening and a stable argsort, i.e. the k
    smallest by (fp32 key, position in the probe concatenation); then the selected rows are
    re-evaluated in fp64 and ordered by _smallest_k."""
    if k < 1:
        raise ValueError(f"k={k} must be >= 1")
    y = np.asarray(query, dtype=np.float64).ravel()
    sizes = np.array([len(a) for a in lists], dtype=np.int64)
    row_ids = np.concatenate(list(lists)).astype(np.int64) if len(lists) else np.empty(0, np.int64)
    vectors32 = np.ascontiguousarray(data.x32[row_ids])
    norms32 = data.sq_norms[row_ids].astype(np.float32)
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    probe = _probe(cent, y, n_probe, 1)
    blocks = [(offsets[c], offsets[c + 1]) for c in probe]
    blocks = [(lo, hi) for lo, hi in blocks if hi > lo]
    if not blocks:
        return np.empty(0, np.int64), np.empty(0, np.float64)
    y32 = y.astype(np.float32)
    d2 = np.concatenate([vectors32[lo:hi] @ y32 for lo, hi in blocks])
    norms = np.concatenate([norms32[lo:hi] for lo, hi in blocks])
    ids = np.concatenate([row_ids[lo:hi] for lo, hi in blocks])
    d2 = norms - np.float32(2.0) * d2
    k_sel = min(k, len(d2))
    if k_sel < len(d2):
        part = np.argpartition(d2, k_sel - 1)[:k_sel]
        boundary = d2[part].max()
        cand = np.flatnonzero(d2 <= boundary)
        order = np.argsort(d2[cand], kind="stable")[:k_sel]
        sel_ids = ids[cand[order]]
    else:
        sel_ids = ids
    ex = data.x64[sel_ids] @ y
    ex *= -2.0
    ex += data.sq_norms[sel_ids]
    ex += float(y @ y)
    np.maximum(ex, 0.0, out=ex)
    return smallest_k(ex, sel_ids, len(sel_ids))
