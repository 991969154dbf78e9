"""Device-resident k-NN / DEANN timings (CUDA events) for A/B runs of the pruned FILTER.

    python scripts/knn_perf.py c3 [--reps 5]     # env: DK_KNN_TMAJOR=0, DK_KNN_PRUNE=0, DK_KNN_STATS=1

Prints one JSON line: per-rep ms of dk_knn and dk_deann (queries, outputs in HBM) and the
FILTER sweep's own time (library events, dk_set_profiling 1).
"""

import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402
from paper_2107_02736_b200 import _lib  # noqa: E402

MAN = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                  "bandwidths.json")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nq", type=int, default=0)
    args = ap.parse_args()
    W = workloads.make(args.config)
    Q = W.Q[: args.nq] if args.nq else W.Q
    h = W.h if W.h is not None else MAN[args.config]["h"]
    ds = g.Dataset.from_array(W.X)
    lib = _lib.load()
    nq, k = Q.shape[0], W.k
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    idx = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    d2 = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    out = torch.empty(nq, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def knn():
        _lib.check(lib.dk_knn(ds.handle, Qd.data_ptr(), nq, k, idx.data_ptr(), d2.data_ptr(), st))

    def deann():
        _lib.check(lib.dk_deann(ds.handle, Qd.data_ptr(), nq, _lib.family_code(W.family), h, k, W.m, 7, 0,
                                out.data_ptr(), None, None, None, st))

    res = {"config": args.config, "nq": nq, "k": k, "m": W.m,
           "env": {v: os.environ.get(v) for v in ("DK_KNN_TMAJOR", "DK_KNN_PRUNE", "DK_KNN_STRIDE")}}
    for name, fn in (("knn", knn), ("deann", deann)):
        fn()
        fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        res[name + "_ms"] = ms
        res[name + "_qps"] = nq / (min(ms) / 1e3)
    _lib.check(lib.dk_set_profiling(ds.handle, 1))
    knn()
    kms, kfl, kby = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.dk_last_kernel_ms(ds.handle, ctypes.byref(kms), ctypes.byref(kfl), ctypes.byref(kby)))
    _lib.check(lib.dk_set_profiling(ds.handle, 0))
    res["filter_ms"] = kms.value
    res["filter_tflops_swept"] = kfl.value / (kms.value / 1e3) / 1e12
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
