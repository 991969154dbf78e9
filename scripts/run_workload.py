"""Run one configuration's hot path a few times (profiling / timing driver).

    python scripts/run_workload.py c2 naive [--reps 3] [--nq N]
    python scripts/run_workload.py c3 deann|knn|naive
    python scripts/run_workload.py c4 naive-exp|naive-lap|deann-exp|deann-lap
    python scripts/run_workload.py c5 naive|deann

Prints one JSON line per op with CUDA-event timings (ms) of each repetition.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402

MAN = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                  "bandwidths.json")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("op")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nq", type=int, default=0)
    args = ap.parse_args()
    t0 = time.perf_counter()
    W = workloads.make(args.config)
    gen_s = time.perf_counter() - t0
    fam = W.family
    key = args.config
    if args.op.endswith("-lap"):
        fam, key = "laplacian", f"{args.config}-laplacian"
    elif args.op.endswith("-exp"):
        fam = "exponential"
    h = W.h if W.h is not None else MAN[key]["h"]
    Q = W.Q[: args.nq] if args.nq else W.Q
    t0 = time.perf_counter()
    ds = g.Dataset.from_array(W.X)
    fit_s = time.perf_counter() - t0
    spec = g.KernelSpec(fam, h)
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    nq = Q.shape[0]
    out = torch.empty(nq, dtype=torch.float64, device="cuda")
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if args.op.startswith("naive"):
            g.naive_kde_into(ds, spec, Qd, out)
        elif args.op.startswith("knn"):
            g.knn_batch(ds, Q, W.k)
        else:
            g.deann_arrays(ds, spec, Q, W.k, W.m, seed=12345)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    stats = None
    if args.op.startswith("naive"):
        import ctypes

        from paper_2107_02736_b200 import _lib

        v = [ctypes.c_int64() for _ in range(4)]
        _lib.check(_lib.load().dk_kde_stats(ds.handle, *[ctypes.byref(x) for x in v]))
        stats = dict(zip(("hybrid_queries", "hybrid_fallbacks", "hot_pairs", "pairs"), (x.value for x in v)))
    if args.op.startswith(("knn", "deann")):
        import ctypes

        from paper_2107_02736_b200 import _lib

        v = [ctypes.c_int64() for _ in range(4)]
        _lib.check(_lib.load().dk_knn_stats(ds.handle, *[ctypes.byref(x) for x in v]))
        qn_, cs, cm, fb = (x.value for x in v)
        stats = {"queries": qn_, "cand_avg": cs / max(qn_, 1), "cand_max": cm, "fallbacks": fb}
    print(json.dumps({"knn_stats": stats, "config": args.config, "op": args.op, "family": fam, "h": h, "nq": nq, "n": W.X.shape[0],
                      "d": W.X.shape[1], "k": W.k, "m": W.m, "ms": times, "qps_best": nq / (min(times) / 1e3),
                      "gen_s": gen_s, "fit_s": fit_s}), flush=True)


if __name__ == "__main__":
    main()
