"""k-NN / DEANN results must not depend on the batch split: run a config with the default batch plan and
with DK_KNN_MAX_BATCH=16384 (the round-1 split) in subprocesses and compare indices, distances and
DEANN values bit for bit.

    python scripts/batch_check.py c5 [nq] [VAR=value ...]     # the second run's environment
    python scripts/batch_check.py c5 0 DK_KNN_GTILES=600      # a looser threshold pass: some queries overflow
                                                              # their candidate lists and take the exact scan
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, nq, out):
    sys.path.insert(0, ROOT)
    import json

    import paper_2107_02736_b200 as g
    import workloads

    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(config)
    ds = g.Dataset.from_array(W.X)
    Q = W.Q[:nq] if nq else W.Q
    idx, d2 = g.knn_batch(ds, Q, W.k)
    vals, nbr, _ = g.deann_arrays(ds, g.KernelSpec(W.family, W.h if W.h is not None else man[config]["h"]), Q, W.k, W.m,
                                  seed=77, export_neighbors=True)
    np.savez(out, idx=idx, d2=d2, vals=vals, nbr=nbr)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        sys.exit(0)
    config = sys.argv[1]
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    outs = []
    alt = dict(a.split("=", 1) for a in sys.argv[3:]) or {"DK_KNN_MAX_BATCH": "16384"}
    for name, env in [("default", {}), ("alt", alt)]:
        out = f"/tmp/batch_check_{name}.npz"
        subprocess.run([sys.executable, __file__, "--child", config, str(nq), out], check=True,
                       env={**os.environ, **env})
        outs.append(np.load(out))
    a, b = outs
    same_idx = np.array_equal(a["idx"], b["idx"])
    same_d2 = np.array_equal(a["d2"], b["d2"])
    same_nbr = np.array_equal(a["nbr"], b["nbr"]) and np.array_equal(a["idx"], a["nbr"])
    same_vals = np.array_equal(a["vals"], b["vals"])
    print(f"{config}: {a['idx'].shape[0]} queries; idx equal {same_idx}, d2 equal {same_d2}, "
          f"deann neighbours equal {same_nbr}, deann values equal {same_vals}")
    sys.exit(0 if (same_idx and same_d2 and same_nbr and same_vals) else 1)
