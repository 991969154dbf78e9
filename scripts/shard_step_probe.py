"""Per-rank step time of dataset-sharded c2 at N = 1, 2, 4, 8 simulated on one GPU.

    python scripts/shard_step_probe.py

Each rank of the N-GPU bench owns n/N rows and runs the same per-step sequence
(query check + encode + sweep + reduce, DK_OUT_SUM); this times that sequence for
a 1/N shard on one B200, which bounds the N-GPU strong-scaling efficiency before
the NCCL all-reduce of the 80 KB partial sums is added.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402


def main():
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make("c2")
    spec = g.KernelSpec("gaussian", man["c2"]["h"])
    n = W.X.shape[0]
    Qd = torch.from_numpy(W.Q).cuda()
    out = torch.empty(len(W.Q), dtype=torch.float64, device="cuda")
    res = {}
    for N in (1, 2, 4, 8):
        ds = g.Dataset.from_array(W.X[: n // N], global_offset=0, global_n=n)
        for _ in range(5):
            g.naive_kde_into(ds, spec, Qd, out, sums=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 200
        e0.record()
        for _ in range(steps):
            g.naive_kde_into(ds, spec, Qd, out, sums=True)
        e1.record()
        e1.synchronize()
        res[N] = e0.elapsed_time(e1) / steps
        ds.free()
    eff = {N: res[1] / (N * res[N]) for N in res}
    print(json.dumps({"ms_per_step": res, "efficiency_without_allreduce": eff}))


if __name__ == "__main__":
    main()
