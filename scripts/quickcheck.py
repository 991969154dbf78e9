"""Quick GPU-vs-oracle check of every C-ABI path (developer tool; not a test)."""

import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from oracle.philox import IndexReplay, NeighborReplay  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def main():
    rng = np.random.default_rng(0)
    for name, X, Q in [
        ("normal", rng.normal(size=(5000, 24)).astype(np.float32), rng.normal(size=(300, 24))),
        ("int", rng.integers(0, 255, size=(7000, 128)).astype(np.float32),
         rng.integers(0, 255, size=(257, 128)).astype(np.float64)),
        ("tiny", rng.normal(size=(3, 2)).astype(np.float32), rng.normal(size=(5, 2))),
    ]:
        t0 = time.time()
        ds = g.Dataset.from_array(X)
        od = O.Data(X)
        print(f"[{name}] fit n={X.shape[0]} d={X.shape[1]} exact={ds.exact_mode} ({time.time()-t0:.2f}s)", flush=True)
        for fam, h in [("gaussian", 3.0 if name != "int" else 300.0), ("exponential", 2.0 if name != "int" else 400.0),
                       ("laplacian", 5.0 if name != "int" else 4000.0)]:
            got = g.naive_kde(ds, g.KernelSpec(fam, h), Q).values
            ref = O.naive_kde(od, fam, h, Q)
            print(f"  naive {fam:12s} max rel {rel(got, ref):.3e}  min ref {ref.min():.3e}", flush=True)
        k = min(10, X.shape[0])
        idx, d2 = g.knn_batch(ds, Q, k)
        bad = 0
        for j in range(Q.shape[0]):
            ri, rd = O.brute_force_knn(od, Q[j], k)
            if not np.array_equal(ri, idx[j]):
                bad += 1
                if bad < 3:
                    print("   knn mismatch", j, ri, idx[j], rd, d2[j])
        print(f"  knn k={k}: {bad} mismatching queries of {Q.shape[0]}", flush=True)
        if X.shape[0] > 20:
            m = 50
            fam, h = "gaussian", (3.0 if name != "int" else 300.0)
            vals, nbr, smp = g.deann_arrays(ds, g.KernelSpec(fam, h), Q, k, m, seed=1234, export_neighbors=True,
                                            export_samples=True)
            worst = 0.0
            for j in range(Q.shape[0]):
                ri, rd = O.brute_force_knn(od, Q[j], k)
                v = O.deann(od, fam, h, NeighborReplay(ri, rd), Q[j], k, m, rng=IndexReplay(1234, j, X.shape[0]))[0]
                worst = max(worst, abs(v - vals[j]) / v)
            print(f"  deann k={k} m={m}: max rel vs oracle replay {worst:.3e}", flush=True)
            est = g.rs_kde(ds, g.KernelSpec(fam, h), Q[0], 64, g.PhiloxSampler(99))
            ref = O.rs_kde(od, fam, h, Q[0], 64, IndexReplay(99, 0, X.shape[0]))
            print(f"  rs m=64: gpu {est.value:.12g} oracle {ref:.12g}", flush=True)


if __name__ == "__main__":
    main()
