"""Pruned vs unpruned k-NN FILTER pass on one configuration (DK_KNN_PRUNE).

    python scripts/prune_check.py c3 [--reps 10] [--nq N]

Each setting runs in its own subprocess; prints the median CUDA-event time of dk_knn and
dk_deann per setting, the first-call (fit incl. clustering) time, and whether the k-NN
indices and distances are identical.
"""

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, reps, nq, out):
    sys.path.insert(0, ROOT)
    import ctypes

    import numpy as np
    import torch

    import paper_2107_02736_b200 as g
    import workloads
    from paper_2107_02736_b200 import _lib

    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(config)
    Q = W.Q[:nq] if nq else W.Q
    ds = g.Dataset.from_array(W.X)
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    n, k = len(Q), W.k
    idx = torch.empty((n, k), dtype=torch.int64, device="cuda")
    d2 = torch.empty((n, k), dtype=torch.float64, device="cuda")
    vals = torch.empty(n, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    h = man[config]["h"] if W.h is None else W.h

    def knn():
        _lib.check(lib.dk_knn(ds.handle, Qd.data_ptr(), n, k, idx.data_ptr(), d2.data_ptr(), st))

    def deann():
        _lib.check(lib.dk_deann(ds.handle, Qd.data_ptr(), n, 0, h, k, W.m, 7, 0, vals.data_ptr(), None, None, None, st))

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    knn()
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    res = {"first_call_s": first}
    for name, fn in (("knn", knn), ("deann", deann)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name + "_ms"] = sorted(ts)[len(ts) // 2]
    knn()
    torch.cuda.synchronize()
    np.save(out + "_idx.npy", idx.cpu().numpy())
    np.save(out + "_d2.npy", d2.cpu().numpy())
    v = [ctypes.c_int64() for _ in range(4)]
    _lib.check(lib.dk_knn_stats(ds.handle, *[ctypes.byref(x) for x in v]))
    res["fallbacks"] = v[3].value
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--child", default="")
    a = ap.parse_args()
    if a.child:
        child(a.config, a.reps, a.nq, a.child)
        return
    import numpy as np

    res = {}
    for setting in ("0", "1"):
        out = f"/tmp/prune_{setting}"
        env = dict(os.environ, DK_KNN_PRUNE=setting, DK_KNN_STATS="1")
        p = subprocess.run([sys.executable, __file__, a.config, "--reps", str(a.reps), "--nq", str(a.nq),
                            "--child", out], env=env, capture_output=True, text=True)
        if p.returncode:
            print(setting, "FAILED", p.stderr[-3000:])
            return
        res["prune" if setting == "1" else "plain"] = json.loads(p.stdout.strip().splitlines()[-1])
        lines = [l for l in p.stderr.splitlines() if l.startswith("[dk]")]
        if lines:
            res["swept_" + setting] = lines[-1]
    same_idx = np.array_equal(np.load("/tmp/prune_0_idx.npy"), np.load("/tmp/prune_1_idx.npy"))
    same_d2 = np.array_equal(np.load("/tmp/prune_0_d2.npy"), np.load("/tmp/prune_1_d2.npy"))
    print(json.dumps({"config": a.config, **res, "identical_idx": bool(same_idx), "identical_d2": bool(same_d2)}))


if __name__ == "__main__":
    main()
