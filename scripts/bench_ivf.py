"""IVF build + probed k-NN + DEANN-with-IVF throughput.

    python scripts/bench_ivf.py [--config c3] [--clusters 1000] [--n-probe 10] [--k 100] [--m 1000]

GPU: ivf_build on the full config dataset, then ivf_query_batch / deann_batch
over the config's queries (wall time around synchronous calls from host arrays,
best of 3 after a full-size warm-up; the build is host-driven k-means++ + device
Lloyd).  CPU: the oracle restatement
of the reference (same algorithm, NumPy/OpenBLAS) on a bounded sample — the
build on a 100k-row subsample with 128 clusters (GPU timed on the same), the
query on 32 queries.  Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402  (CPU baseline only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--clusters", type=int, default=1000)
    ap.add_argument("--n-probe", type=int, default=10)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--m", type=int, default=1000)
    args = ap.parse_args()
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(args.config)
    h = W.h if W.h is not None else man[args.config]["h"]
    ds = g.Dataset.from_array(W.X)
    Q = np.ascontiguousarray(W.Q)
    out = {"config": args.config, "n": ds.n, "d": ds.d, "nq": len(Q), "n_clusters": args.clusters,
           "n_probe": args.n_probe, "k": args.k}
    t0 = time.perf_counter()
    index = g.ivf_build(ds, args.clusters, seed=0)
    out["gpu_build_s"] = time.perf_counter() - t0
    ann = g.IvfAnnIndex(ds, index, args.n_probe)
    ann.query_batch(Q, args.k)  # full-size warm-up (scratch buffers grow once)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        idx, d2, cnt = ann.query_batch(Q, args.k)
        ts.append(time.perf_counter() - t0)
    out["gpu_query_s"] = min(ts)
    out["gpu_query_qps"] = len(Q) / out["gpu_query_s"]
    sizes = np.array([len(a) for a in index.assignments])
    out["list_size_mean"], out["list_size_max"] = float(sizes.mean()), int(sizes.max())
    exact_i, _ = g.knn_batch(ds, Q[:256], args.k)
    out["recall_at_k_256q"] = float(np.mean([len(np.intersect1d(idx[j, :cnt[j]], exact_i[j])) / args.k
                                             for j in range(256)]))
    spec = g.KernelSpec(W.family, h)
    g.deann_batch(ds, spec, ann, Q, args.k, args.m, rng=g.PhiloxSampler(1))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        g.deann_batch(ds, spec, ann, Q, args.k, args.m, rng=g.PhiloxSampler(1))
        ts.append(time.perf_counter() - t0)
    out["gpu_deann_ivf_qps"] = len(Q) / min(ts)
    # bounded CPU sample: oracle (reference algorithm) vs GPU on a 100k x d subsample, 128 clusters
    sub = W.X[:100_000]
    dsub = g.Dataset.from_array(sub)
    t0 = time.perf_counter()
    g.ivf_build(dsub, 128, seed=0)
    out["gpu_build_100k_128_s"] = time.perf_counter() - t0
    od = O.Data(sub)
    t0 = time.perf_counter()
    cent, lists = O.ivf_build(od, 128, 0)
    out["cpu_build_100k_128_s"] = time.perf_counter() - t0
    odf = O.Data(W.X)
    oc, ol = index.centroids, index.assignments
    t0 = time.perf_counter()
    for j in range(32):
        O.ivf_query(odf, oc, ol, Q[j], args.k, args.n_probe, formula=1)
    out["cpu_query_qps_32q"] = 32 / (time.perf_counter() - t0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
