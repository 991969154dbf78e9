"""A/B timing of alternative builds of the C-ABI library on one workload.

    python scripts/ab_libs.py c2 variants/lib_a.so variants/lib_b.so ... [--reps 30] [--rounds 2]

Each library runs in its own subprocess (DK_LIBRARY=<path>); rounds interleave the
libraries so clock drift hits all of them alike.  Prints the median kernel-call
time per library and the max relative difference of its KDE values against the
first library's.
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, op, reps, out_path):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import paper_2107_02736_b200 as g
    import workloads

    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(config)
    fam = {"naive-exp": "exponential", "naive-lap": "laplacian", "deann-exp": "exponential",
           "deann-lap": "laplacian"}.get(op, W.family)
    key = f"{config}-laplacian" if fam == "laplacian" else config
    h = man[key]["h"] if fam == "laplacian" or W.h is None else W.h
    ds = g.Dataset.from_array(W.X)
    spec = g.KernelSpec(fam, h)
    Qd = torch.from_numpy(np.ascontiguousarray(W.Q)).cuda()
    out = torch.empty(W.Q.shape[0], dtype=torch.float64, device="cuda")
    if op.startswith("deann"):
        k, m = (50, 500) if config == "c4" else (100, 1000)
        vals = torch.empty(len(W.Q), dtype=torch.float64, device="cuda")
        fam_code = _lib_family = {"gaussian": 0, "exponential": 1, "laplacian": 2}[fam]

        def call():
            from paper_2107_02736_b200 import _lib
            _lib.check(_lib.load().dk_deann(ds.handle, Qd.data_ptr(), len(W.Q), fam_code, h, k, m, 12345, 0,
                                            vals.data_ptr(), None, None, None,
                                            torch.cuda.current_stream().cuda_stream))
        out = vals
    elif op == "knn":
        from paper_2107_02736_b200 import _lib

        k = 100
        idx = torch.empty((len(W.Q), k), dtype=torch.int64, device="cuda")
        d2 = torch.empty((len(W.Q), k), dtype=torch.float64, device="cuda")

        def call():
            _lib.check(_lib.load().dk_knn(ds.handle, Qd.data_ptr(), len(W.Q), k, idx.data_ptr(), d2.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    else:
        def call():
            g.naive_kde_into(ds, spec, Qd, out)
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
    np.save(out_path, (d2 if op == "knn" else out).cpu().numpy().ravel())
    print(json.dumps({"ms": sorted(ts)[len(ts) // 2], "min": min(ts)}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--op", default="naive")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--child", default="")
    args = ap.parse_args()
    if args.child:
        child(args.config, args.op, args.reps, args.child)
        return
    import numpy as np

    res = {lib: [] for lib in args.libs}
    for r in range(args.rounds):
        for i, lib in enumerate(args.libs):
            outp = f"/tmp/ab_{i}.npy"
            env = dict(os.environ, DK_LIBRARY=os.path.abspath(lib))
            p = subprocess.run([sys.executable, __file__, args.config, lib, "--op", args.op, "--reps", str(args.reps),
                                "--child", outp], env=env, capture_output=True, text=True)
            if p.returncode != 0:
                print(lib, "FAILED", p.stderr[-2000:])
                continue
            res[lib].append(json.loads(p.stdout.strip().splitlines()[-1]))
    base = np.load("/tmp/ab_0.npy")
    for i, lib in enumerate(args.libs):
        v = np.load(f"/tmp/ab_{i}.npy")
        rel = float(np.max(np.abs(v - base) / np.maximum(np.abs(base), 1e-300)))
        print(json.dumps({"lib": os.path.basename(lib), "ms": [x["ms"] for x in res[lib]],
                          "min": [x["min"] for x in res[lib]], "max_rel_vs_first": rel}))


if __name__ == "__main__":
    main()
