"""Randomised GPU-vs-oracle parity sweep over the exact KDE, k-NN, RS and DEANN paths.

Developer tool (not a test): `python scripts/fuzz.py [seconds] [first_seed]` draws
dataset shapes, value distributions, kernel families, k and m at random until the
time budget is spent and prints one line per trial; it exits 1 if any trial broke
a north-star gate (exact KDE 1e-4 relative, k-NN sets equal up to ties within
1e-6 relative, RS / DEANN 1e-5 relative on the same indices).
"""

import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from paper_2107_02736_b200 import _lib  # noqa: E402
from oracle.philox import IndexReplay, NeighborReplay  # noqa: E402


def make_rows(rng, kind, n, d):
    if kind == "normal":
        return rng.normal(size=(n, d)) * rng.choice([0.1, 1.0, 30.0])
    if kind == "mixture":
        c = int(rng.integers(2, 60))
        means = rng.normal(size=(c, d)) * rng.choice([1.0, 4.0, 10.0])
        return means[rng.integers(0, c, size=n)] + rng.normal(size=(n, d)) * rng.choice([0.05, 0.3, 1.0])
    if kind == "integer":
        return rng.integers(0, int(rng.choice([2, 16, 256])), size=(n, d)).astype(np.float64)
    if kind == "sparse":
        return np.where(rng.random((n, d)) < 0.8, 0.0, rng.random((n, d)))
    if kind == "unit":
        x = rng.normal(size=(n, d)) + rng.normal(size=(1, d)) * rng.choice([0.0, 2.0])
        return x / np.maximum(np.linalg.norm(x, axis=1, keepdims=True), 1e-30)
    if kind == "pool":  # few distinct rows: many exact ties
        pool = rng.integers(-3, 4, size=(int(rng.integers(1, 40)), d)).astype(np.float64)
        return pool[rng.integers(0, pool.shape[0], size=n)]
    if kind == "offset":
        return rng.normal(size=(n, d)) + 100.0
    raise ValueError(kind)


KINDS = ["normal", "mixture", "integer", "sparse", "unit", "pool", "offset"]


def tie_tolerant_equal(gi, gd, ri, rd, noise=0.0):
    """Index sets equal up to rows whose distance is within 1e-6 relative of the boundary.

    `noise`: absolute rounding level of the reference's own distances (norms identity in fp64,
    ~64 ulp of |q|^2 + |x|^2), below which its order of two rows is not meaningful."""
    if np.array_equal(gi, ri):
        return True
    bound = rd[-1]
    tol = 1e-6 * max(bound, 1e-300) + noise
    only_g = np.setdiff1d(gi, ri)
    only_r = np.setdiff1d(ri, gi)
    gpos = {int(v): i for i, v in enumerate(gi)}
    rpos = {int(v): i for i, v in enumerate(ri)}
    if any(abs(gd[gpos[int(v)]] - bound) > tol for v in only_g):
        return False
    if any(abs(rd[rpos[int(v)]] - bound) > tol for v in only_r):
        return False
    # common rows may be permuted only among (near-)equal distances
    return bool(np.all(np.abs(np.sort(gd) - np.sort(rd)) <= 1e-6 * np.maximum(np.sort(rd), 1e-300) + noise + 1e-300))


def gen(seed):
    """The trial's inputs: (rng, kind, n, d, nq, X, Q, family, h, scale)."""
    rng = np.random.default_rng(seed)
    kind = KINDS[int(rng.integers(0, len(KINDS)))]
    size = rng.choice(["small", "mid", "big", "hyb"], p=[0.3, 0.4, 0.2, 0.1])
    if size == "small":
        n = int(rng.integers(1, 400))
    elif size == "mid":
        n = int(rng.integers(400, 30000))
    elif size == "big":
        n = int(rng.integers(66000, 260000))
    else:  # large gaussian batches on non-integer rows: the two-precision exact KDE
        n = int(rng.integers(131072, 400000))
        kind = str(rng.choice(["normal", "mixture", "sparse", "unit", "offset"]))
    d = int(rng.choice([1, 2, 3, 7, 16, 31, 64, 96, 100, 128, 129, 200, 300, 784]))
    if size in ("big", "hyb"):
        d = min(d, 128)
    nq = int(rng.choice([1, 2, 33, 128, 129, 300, 700, 2500]))
    if size == "big":
        nq = min(nq, 700)
    if size == "hyb":
        nq = int(rng.choice([2048, 2500, 4097]))
    X = make_rows(rng, kind, n, d).astype(np.float32)
    Q = make_rows(rng, kind, nq, d)
    if rng.random() < 0.3:  # queries on data points
        take = rng.integers(0, n, size=nq)
        Q = X[take].astype(np.float64)
    fam = str(rng.choice(["gaussian", "exponential", "laplacian"])) if size != "hyb" else "gaussian"
    if fam == "laplacian" and n * nq * d > 4e10:
        fam = "gaussian"
    # bandwidth from a pilot so that values neither underflow nor saturate
    a = X[rng.integers(0, n, size=200)].astype(np.float64)
    b = Q[rng.integers(0, nq, size=200)]
    if fam == "laplacian":
        scale = float(np.median(np.abs(a - b).sum(1)))
    else:
        scale = float(np.median(np.sqrt(((a - b) ** 2).sum(1))))
    scale = max(scale, 0.5)
    h = scale * float(rng.choice([0.15, 0.4, 1.0, 3.0]))
    return rng, kind, n, d, nq, X, Q, fam, h, scale


def trial(seed):
    rng, kind, n, d, nq, X, Q, fam, h, scale = gen(seed)
    spec = g.KernelSpec(fam, h)
    ds = g.Dataset.from_array(X)
    od = O.Data(X)
    msgs = []
    ok = True

    chk = np.arange(nq) if float(n) * nq * d < 3e10 else np.sort(rng.choice(nq, size=64, replace=False))
    got = g.naive_kde(ds, spec, Q).values[chk]
    ref = O.naive_kde(od, fam, h, Q[chk])
    live = ref > 1e-280
    e_naive = float(np.max(np.abs(got[live] - ref[live]) / ref[live])) if live.any() else 0.0
    dead = float(np.max(np.abs(got[~live]))) if (~live).any() else 0.0
    if e_naive > 1e-4 or dead > 1e-270:
        ok = False
        msgs.append(f"NAIVE {e_naive:.2e} dead {dead:.1e}")

    redo = ctypes.c_int64(0)
    _lib.check(_lib.load().dk_kde_redo_count(ds.handle, ctypes.byref(redo)))
    xn_max = float(od.sq_norms.max())
    k = int(min(n, rng.choice([1, 5, 50, 100, 257])))
    nchk = min(nq, 48)
    sel = rng.choice(nq, size=nchk, replace=False) if nq > nchk else np.arange(nq)
    gi, gd = g.knn_batch(ds, Q, k)
    exact_same = 0
    e_d2 = 0.0
    for j in sel:
        ri, rd = O.brute_force_knn(od, Q[j], k)
        if np.array_equal(ri, gi[j]):
            exact_same += 1
        elif not tie_tolerant_equal(gi[j], gd[j], ri, rd, noise=64 * 2.2e-16 * (float(Q[j] @ Q[j]) + xn_max)):
            ok = False
            msgs.append(f"KNN q{j}")
        # the reference's d2 (norms identity in fp64) carries ~4 ulp of |q|^2 + |x|^2: floor the denominator there
        floor = 4e-9 * (float(Q[j] @ Q[j]) + xn_max) + 1e-300
        e_d2 = max(e_d2, float(np.max(np.abs(np.sort(gd[j]) - np.sort(rd)) / np.maximum(np.sort(rd), floor))))
    if e_d2 > 1e-6:
        ok = False
        msgs.append(f"KNN-D2 {e_d2:.2e}")

    e_deann = 0.0
    if n > k:
        m = int(rng.choice([1, 17, 500, 2000]))
        kk = int(rng.choice([0, k]))
        seed_s = int(rng.integers(0, 2**31))
        vals, nbr, _ = g.deann_arrays(ds, spec, Q, kk, m, seed=seed_s, export_neighbors=True)
        for j in sel:
            if kk:
                xi = np.asarray(nbr[j], dtype=np.int64)
                rd = O.batch_sqdist(Q[j].reshape(1, -1), od.x64[xi], od.sq_norms[xi])[0]
                nr = NeighborReplay(xi, rd)
            else:
                nr = None
            want = O.deann(od, fam, h, nr, Q[j], kk, m, rng=IndexReplay(seed_s, int(j), n))[0]
            if want > 1e-280:
                e_deann = max(e_deann, abs(vals[j] - want) / want)
            elif abs(vals[j]) > 1e-270:
                e_deann = np.inf
        if e_deann > 1e-5:
            ok = False
            msgs.append(f"DEANN {e_deann:.2e} (k={kk}, m={m})")
    ds.free()
    print(f"seed {seed:6d} {'ok ' if ok else 'BAD'} {kind:8s} n={n:7d} d={d:4d} nq={nq:5d} {fam:11s} h={h:9.3g} k={k:4d} "
          f"naive {e_naive:.1e} redo {redo.value} knn same {exact_same}/{len(sel)} d2 {e_d2:.1e} deann {e_deann:.1e} {' '.join(msgs)}", flush=True)
    return ok


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    t0 = time.time()
    bad = 0
    count = 0
    while time.time() - t0 < budget:
        try:
            if not trial(seed):
                bad += 1
        except Exception as exc:  # a crash is a finding too
            bad += 1
            print(f"seed {seed:6d} EXC {type(exc).__name__}: {exc}", flush=True)
        seed += 1
        count += 1
    print(f"fuzz: {count} trials, {bad} bad")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
