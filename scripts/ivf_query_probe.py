"""Build a c3 IVF index and run one batched probed query (for ncu launch lists).

    python scripts/ivf_query_probe.py [--clusters 1000] [--n-probe 10] [--k 100] [--nq 10000]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clusters", type=int, default=1000)
    ap.add_argument("--n-probe", type=int, default=10)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--nq", type=int, default=10000)
    args = ap.parse_args()
    W = workloads.make("c3")
    ds = g.Dataset.from_array(W.X)
    index = g.ivf_build(ds, args.clusters, seed=0)
    ann = g.IvfAnnIndex(ds, index, args.n_probe)
    Q = np.ascontiguousarray(W.Q[: args.nq])
    ann.query_batch(Q[:64], args.k)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        ann.query_batch(Q, args.k)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"nq": len(Q), "query_ms": [round(1e3 * t, 3) for t in ts]}))


if __name__ == "__main__":
    main()
