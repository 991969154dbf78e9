"""End-to-end time of one c3 exact-KDE call through the public API (pinned host queries in,
values out; the two-precision path):

    python scripts/e2e_c3_exact.py
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


def main():
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make("c3")
    ds = g.Dataset.from_array(W.X)
    spec = g.KernelSpec("gaussian", man["c3"]["h"])
    Qh = torch.from_numpy(W.Q).pin_memory().numpy()
    for _ in range(5):
        g.naive_kde(ds, spec, Qh)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        g.naive_kde(ds, spec, Qh).values
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"c3_e2e_ms": 1e3 * float(np.median(ts))}))


if __name__ == "__main__":
    main()
