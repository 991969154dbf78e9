"""Run the naive KDE sweep back to back for a few seconds and sample SM clock, power
and throttle reasons through NVML (is the epilogue-heavy sweep power-capped?).

    python scripts/power_probe.py c2 [--seconds 3] [--op naive|naive-exp]
"""

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--op", default="naive")
    args = ap.parse_args()
    man = json.load(open(os.path.join(ROOT, "tests", "golden", "bandwidths.json")))
    W = workloads.make(args.config)
    fam = "exponential" if args.op == "naive-exp" else W.family
    h = W.h if W.h is not None else man[args.config]["h"]
    ds = g.Dataset.from_array(W.X)
    spec = g.KernelSpec(fam, h)
    Qd = torch.from_numpy(np.ascontiguousarray(W.Q)).cuda()
    out = torch.empty(W.Q.shape[0], dtype=torch.float64, device="cuda")
    g.naive_kde_into(ds, spec, Qd, out)
    torch.cuda.synchronize()
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(hd) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hd)))
            time.sleep(0.01)

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + args.seconds
    calls = 0
    e0.record()
    while time.time() < t_end:
        for _ in range(20):
            g.naive_kde_into(ds, spec, Qd, out)
        calls += 20
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    stop.set()
    th.join()
    clk = np.array([s[0] for s in samples])
    pw = np.array([s[1] for s in samples])
    reasons = 0
    for s in samples:
        reasons |= s[2]
    print(json.dumps({"config": args.config, "op": args.op, "ms_per_call": e0.elapsed_time(e1) / calls,
                      "sm_mhz_median": float(np.median(clk)), "sm_mhz_min": int(clk.min()),
                      "power_w_median": float(np.median(pw)), "power_w_max": float(pw.max()),
                      "power_limit_w": pynvml.nvmlDeviceGetEnforcedPowerLimit(hd) / 1000.0,
                      "throttle_reasons_or": hex(reasons), "samples": len(samples)}))


if __name__ == "__main__":
    main()
