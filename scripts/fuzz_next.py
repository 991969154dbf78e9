"""Randomised GPU-vs-oracle sweep over the "next" rows: the permuted sampler (RSP / DEANNP, f1) and the
inverted-file index (f3).  Developer tool: `python scripts/fuzz_next.py [seconds] [first_seed]`.

RSP / DEANNP: values 1e-10 relative, cursors and sample counts exact.  IVF: the build's lists equal
the oracle's, ivf_query_batch's rows equal ivf_query's (ties to the lower row), distances 1e-9.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import fuzz  # noqa: E402
import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402


def trial(seed):
    rng = np.random.default_rng(seed)
    kind = str(rng.choice(["normal", "mixture", "integer", "sparse", "unit", "pool"]))
    n = int(rng.choice([3, 50, 700, 5000, 30000]))
    d = int(rng.choice([1, 3, 8, 24, 100]))
    nq = int(rng.choice([1, 7, 40]))
    X = fuzz.make_rows(rng, kind, n, d).astype(np.float32)
    Q = fuzz.make_rows(rng, kind, nq, d)
    fam = str(rng.choice(["gaussian", "exponential", "laplacian"]))
    a, b = X[rng.integers(0, n, 100)].astype(np.float64), Q[rng.integers(0, nq, 100)]
    scale = max(0.5, float(np.median(np.abs(a - b).sum(1) if fam == "laplacian" else np.sqrt(((a - b) ** 2).sum(1)))))
    h = scale * float(rng.choice([0.4, 1.0, 3.0]))
    ds, od = g.Dataset.from_array(X), O.Data(X)
    spec = g.KernelSpec(fam, h)
    msgs = []
    # --- permuted sampler: shared cursor through a batch
    k = int(min(n - 1, rng.choice([0, 1, 10, 60]))) if n > 1 else 0
    m = int(rng.choice([1, 30, 400]))
    pseed, cur = int(rng.integers(0, 1000)), int(rng.integers(0, n))
    st = g.RspState.from_dataset(ds, pseed, cursor=cur)
    ost = O.Permuted(od, pseed, cursor=cur)
    got = g.deann_batch(ds, spec, g.BruteForceIndex(ds), Q, k, m, rsp_state=st)
    e_rsp = 0.0
    for j in range(nq):
        ref = O.deann_rsp(od, fam, h, lambda y, kk: O.brute_force_knn(od, y, kk), Q[j], k, m, ost)
        if ref[0] > 1e-280:
            e_rsp = max(e_rsp, abs(got[j].value - ref[0]) / ref[0])
    if e_rsp > 1e-10:
        msgs.append(f"RSP {e_rsp:.2e}")
    if st.cursor != ost.cursor:
        msgs.append(f"CURSOR {st.cursor} != {ost.cursor}")
    # --- inverted file
    e_ivf = 0.0
    if n >= 50:
        C = int(min(n // 4, rng.choice([1, 4, 32, 64])))
        p = int(min(C, rng.choice([1, 2, 8])))
        kk = int(min(n, rng.choice([1, 10, 100])))
        iseed = int(rng.integers(0, 1000))
        index = g.ivf_build(ds, C, iseed)
        cent, lists = O.ivf_build(od, C, iseed)
        if not all(x.shape == y.shape and (x == y).all() for x, y in zip(index.assignments, lists)):
            msgs.append("IVF-LISTS")
        else:
            idx, d2, cnt = g.ivf_query_batch(index, ds, Q, kk, p)
            for j in range(nq):
                ri, rd = O.ivf_query(od, cent, lists, Q[j], kk, p)
                if cnt[j] != len(ri) or not np.array_equal(idx[j, :cnt[j]], ri):
                    if not fuzz.tie_tolerant_equal(idx[j, :cnt[j]], d2[j, :cnt[j]], ri, rd,
                                                   noise=64 * 2.2e-16 * (float(Q[j] @ Q[j]) + float(od.sq_norms.max()))):
                        msgs.append(f"IVF q{j}")
                else:
                    e_ivf = max(e_ivf, float(np.max(np.abs(d2[j, :cnt[j]] - rd) / np.maximum(rd, 1e-9 * scale * scale + 1e-300))))
            if e_ivf > 1e-6:
                msgs.append(f"IVF-D2 {e_ivf:.2e}")
    ds.free()
    ok = not msgs
    print(f"seed {seed:6d} {'ok ' if ok else 'BAD'} {kind:8s} n={n:6d} d={d:4d} nq={nq:3d} {fam:11s} k={k:3d} m={m:4d} "
          f"rsp {e_rsp:.1e} ivf {e_ivf:.1e} {' '.join(msgs)}", flush=True)
    return ok


if __name__ == "__main__":
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    t0, bad, count = time.time(), 0, 0
    while time.time() - t0 < budget:
        try:
            bad += 0 if trial(seed) else 1
        except Exception as exc:
            bad += 1
            print(f"seed {seed:6d} EXC {type(exc).__name__}: {exc}", flush=True)
        seed += 1
        count += 1
    print(f"fuzz_next: {count} trials, {bad} bad")
    sys.exit(1 if bad else 0)
