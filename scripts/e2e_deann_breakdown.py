"""Where the end-to-end (host buffers) time of one c3 DEANN batch goes.

    python scripts/e2e_deann_breakdown.py
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
from paper_2107_02736_b200 import _lib  # noqa: E402


def timeit(fn, reps=20):
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
    W = workloads.make("c3")
    h = man["c3"]["h"]
    ds = g.Dataset.from_array(W.X)
    spec = g.KernelSpec("gaussian", h)
    lib = _lib.load()
    Qpin = torch.from_numpy(W.Q).pin_memory()
    Qh = Qpin.numpy()
    Qd = Qpin.cuda()
    nq = len(Qh)
    outd = torch.empty(nq, dtype=torch.float64, device="cuda")
    outh = torch.empty(nq, dtype=torch.float64).pin_memory()
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

    def call(q, o):
        _lib.check(lib.dk_deann(ds.handle, _lib.ptr(q), nq, 0, h, 100, 1000, 7, 0, _lib.ptr(o), None, None, None,
                                st()))

    bf = g.BruteForceIndex(ds)
    r = {
        "device_in_device_out": timeit(lambda: call(Qd, outd)),
        "pinned_in_device_out": timeit(lambda: call(Qh, outd)),
        "device_in_pinned_out": timeit(lambda: call(Qd, outh.numpy())),
        "pinned_in_pinned_out": timeit(lambda: call(Qh, outh.numpy())),
        "deann_arrays_pinned": timeit(lambda: g.deann_arrays(ds, spec, Qh, 100, 1000, seed=7)),
        "deann_batch_pinned": timeit(lambda: g.deann_batch(ds, spec, bf, Qh, 100, 1000, rng=g.PhiloxSampler(7))),
        "h2d_8MB_pinned": timeit(lambda: Qd.copy_(Qpin, non_blocking=True)),
    }
    print(json.dumps({k: round(v, 4) for k, v in r.items()}))


if __name__ == "__main__":
    main()
