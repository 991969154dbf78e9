"""Where the end-to-end (host buffers) time of one c2 naive-KDE call goes.

    python scripts/e2e_breakdown.py
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


def main():
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make("c2")
    ds = g.Dataset.from_array(W.X)
    spec = g.KernelSpec("gaussian", man["c2"]["h"])
    Qpin = torch.from_numpy(W.Q).pin_memory()
    Qh = Qpin.numpy()
    Qpage = np.array(W.Q)
    Qd = Qpin.cuda()
    outd = torch.empty(len(Qh), dtype=torch.float64, device="cuda")
    outh = torch.empty(len(Qh), dtype=torch.float64).pin_memory()
    r = {
        "device_in_device_out": timeit(lambda: g.naive_kde_into(ds, spec, Qd, outd)),
        "device_in_pinned_out": timeit(lambda: g.naive_kde_into(ds, spec, Qd, outh.numpy())),
        "pinned_in_device_out": timeit(lambda: g.naive_kde_into(ds, spec, Qh, outd)),
        "pinned_in_pinned_out": timeit(lambda: g.naive_kde_into(ds, spec, Qh, outh.numpy())),
        "naive_kde_pinned": timeit(lambda: g.naive_kde(ds, spec, Qh)),
        "naive_kde_pageable": timeit(lambda: g.naive_kde(ds, spec, Qpage)),
        "h2d_10MB_pinned": timeit(lambda: Qd.copy_(Qpin, non_blocking=True)),
    }
    print(json.dumps({k: round(v, 4) for k, v in r.items()}))


if __name__ == "__main__":
    main()
