"""A/B of the 2-CTA pair mode (DK_PAIR) on one workload's k-NN / DEANN path.

    python scripts/pair_probe.py c3 knn|deann [--reps 10]

Runs each setting in its own subprocess (DK_PAIR is read when a dataset is fitted),
prints the median CUDA-event time per setting and whether the outputs are identical.
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, op, reps, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import paper_2107_02736_b200 as g
    import workloads
    from paper_2107_02736_b200 import _lib

    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(config)
    ds = g.Dataset.from_array(W.X)
    Qd = torch.from_numpy(np.ascontiguousarray(W.Q)).cuda()
    nq, k = len(W.Q), W.k
    idx = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    d2 = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    vals = torch.empty(nq, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream

    def call():
        if op == "knn":
            _lib.check(lib.dk_knn(ds.handle, Qd.data_ptr(), nq, k, idx.data_ptr(), d2.data_ptr(), st))
        else:
            _lib.check(lib.dk_deann(ds.handle, Qd.data_ptr(), nq, 0, man[config]["h"], k, W.m, 7, 0, vals.data_ptr(),
                                    idx.data_ptr(), None, None, st))

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    np.save(out, idx.cpu().numpy())
    print(json.dumps({"ms": sorted(ts)[len(ts) // 2], "min": min(ts)}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("op")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--child", default="")
    a = ap.parse_args()
    if a.child:
        child(a.config, a.op, a.reps, a.child)
        return
    import numpy as np

    res = {}
    for rnd in range(2):
        for pair in ("0", "1"):
            out = f"/tmp/pair_{pair}.npy"
            env = dict(os.environ, DK_PAIR=pair)
            p = subprocess.run([sys.executable, __file__, a.config, a.op, "--reps", str(a.reps), "--child", out],
                               env=env, capture_output=True, text=True)
            if p.returncode:
                print(pair, "FAILED", p.stderr[-2000:])
                continue
            res.setdefault(pair, []).append(json.loads(p.stdout.strip().splitlines()[-1])["ms"])
    same = np.array_equal(np.load("/tmp/pair_0.npy"), np.load("/tmp/pair_1.npy"))
    print(json.dumps({"config": a.config, "op": a.op, "ms_single": res.get("0"), "ms_pair": res.get("1"),
                      "identical_indices": bool(same)}))


if __name__ == "__main__":
    main()
