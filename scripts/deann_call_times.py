"""Per-call wall times of c3 DEANN through `deann_batch` (pinned host queries, list of Estimates):

    python scripts/deann_call_times.py [calls]

Shows warm-up and outlier calls that a mean over a timed window includes and a median hides.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402


def main():
    calls = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make("c3")
    ds = g.Dataset.from_array(W.X)
    spec = g.KernelSpec("gaussian", man["c3"]["h"])
    Qh = torch.from_numpy(W.Q).pin_memory().numpy()
    bf = g.BruteForceIndex(ds)
    ts = []
    for i in range(calls):
        t0 = time.perf_counter()
        est = g.deann_batch(ds, spec, bf, Qh, W.k, W.m, rng=g.PhiloxSampler(1234 + i))
        est.values
        ts.append(round(1e3 * (time.perf_counter() - t0), 3))
    print(json.dumps(ts))


if __name__ == "__main__":
    main()
