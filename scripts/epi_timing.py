"""Wait accounting of the tile sweep (debug build with -DDK_TIMING, see tile_kernel.cuh).

    DK_LIBRARY=variants/lib_timing.so python scripts/epi_timing.py c2 [naive|knn]

Prints, per sweep call, the share of epilogue time spent waiting for accumulators
(tfull) and column norms (xfull), and the MMA warp's waits on free accumulators
(tempty: epilogue-bound) and on loaded stages (full: feed-bound).
"""

import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
from paper_2107_02736_b200 import _lib  # noqa: E402
import workloads  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    op = sys.argv[2] if len(sys.argv) > 2 else "naive"
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(cfg)
    h = W.h if W.h is not None else man[cfg]["h"]
    ds = g.Dataset.from_array(W.X)
    lib = _lib.load()
    lib.dk_debug_counters.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(8, dtype=np.uint64)
    Qd = torch.from_numpy(np.ascontiguousarray(W.Q)).cuda()
    out = torch.empty(len(W.Q), dtype=torch.float64, device="cuda")
    spec = g.KernelSpec(W.family, h)
    for rep in range(3):
        lib.dk_debug_counters(buf.ctypes.data, 1)
        if op == "naive":
            g.naive_kde_into(ds, spec, Qd, out)
        else:
            g.knn_batch(ds, W.Q, 100)
        torch.cuda.synchronize()
        lib.dk_debug_counters(buf.ctypes.data, 1)
        b = buf.astype(np.float64)
        busy = b[2]
        print(json.dumps({"config": cfg, "op": op, "rep": rep,
                          "epi_tfull_wait_frac": b[0] / busy, "epi_xfull_wait_frac": b[1] / busy,
                          "epi_cycles_per_warp": busy / (148 * 16), "tiles_per_warp": b[6] / (148 * 16),
                          "mma_tempty_wait_per_sm": b[3] / 148, "mma_full_wait_per_sm": b[4] / 148,
                          "producer_empty_wait_per_sm": b[5] / 148}))


if __name__ == "__main__":
    main()
