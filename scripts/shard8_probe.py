"""One rank's step of 8-way dataset-sharded c2 (125k rows, 10k queries), for launch lists."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402

man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
W = workloads.make("c2")
spec = g.KernelSpec("gaussian", man["c2"]["h"])
n = W.X.shape[0]
ds = g.Dataset.from_array(W.X[: n // 8], global_offset=0, global_n=n)
Qd = torch.from_numpy(W.Q).cuda()
out = torch.empty(len(W.Q), dtype=torch.float64, device="cuda")
for _ in range(8):
    g.naive_kde_into(ds, spec, Qd, out, sums=True)
torch.cuda.synchronize()
