"""Benchmark: KDE queries/s — exact (headline, config 2) and DEANN (configs 3 and 5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline step = one exact naive-KDE pass (gaussian, h by the median-1e-3 rule) of all
10,000 queries over the n = 1,000,000 x 128 integer dataset of config 2 — the
"single-GPU fused distance-GEMM + exp + row-sum" workload BASELINE.json names.
N > 1 (torchrun, or `--gpus N` which re-launches itself under torchrun): the same
workload dataset-sharded — each rank fits n/N rows, per-query partial sums, NCCL
all-reduce (fp64 sum) -> strong scaling.

Rank 0 prints ONE JSON line.  Besides the contract keys (`value` device-timed with
inputs in HBM, `e2e` through the public `naive_kde` API with pinned host queries,
`roofline`, `cpu_baseline`, `clocks`, `gpu_launches`) it carries two first-class
objects for the rest of BASELINE's metric ("exact & DEANN at n = 1M-8M"):
  deann  config 3 DEANN (exact k = 100 NN + m = 1,000 Philox samples): device value,
         e2e through `deann_batch` (pinned host queries, list of Estimates), per-kernel
         rooflines, clocks, oracle parity of the timed output, CPU baseline.
  c3_exact  config 3 exact KDE (non-integer rows): the two-precision path (single-pass fp16
         sweep of every pair, split3 sweep of the hot tile halves, per-query bound), its 1x
         roofline fraction, the split3-only time beside it, e2e, parity, CPU baseline.
  c5     config 5 (n = 8M, 100,000 queries): exact KDE and DEANN (k = 100, m = 2,000);
         dataset-sharded over the ranks when N > 1 (all-reduce of partial sums,
         all-gather + merge of per-shard top-k, shared Philox stream).
`--impl reference` times the oracle port (the reference's own CPU algorithm, all host
threads) on the headline config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "KDE queries/sec (exact naive KDE, gaussian) at n=1M, d=128"
UNIT = "queries/s"
WORKLOAD = "c2: exact naive gaussian KDE, n=1,000,000 x d=128 integer rows, 10,000 queries, h by median-1e-3 rule"
# --workload c5: the north star's scale-out config (BASELINE configs[4]), exact KDE part
WORKLOADS = {
    "c2": {"metric": METRIC, "desc": WORKLOAD, "dtype": "fp16-exact-int (fp32 accumulate, fp64 row sums)",
           "l2": "inputs larger than L2 (256 MB fp16 operand + 512 MB fp32 rows > 126 MB)",
           "traffic": "c2_kde_gauss"},
    "c5": {"metric": "KDE queries/sec (exact naive KDE, gaussian) at n=8M, d=96",
           "desc": "c5: exact naive gaussian KDE, n=8,000,000 x d=96 mixture rows (Dirichlet weights), "
                   "100,000 queries, h by median-1e-3 rule",
           "dtype": "fp16 split3 (fp32 accumulate, fp64 row sums)",
           "l2": "inputs larger than L2 (5.1 GB split3 operand + 3.07 GB fp32 rows > 126 MB)",
           "traffic": None},
}


def _peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return {"hbm_gbs": p.get("hbm_gbs", 6650.0), "bf16_tflops": p.get("bf16_tflops", 1590.0),
                "sm_max_mhz": p.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "source": "fallback"}


class ClockSampler:
    """SM clock and throttle reasons sampled every ~5 ms during the timed region (NVML;
    nvidia-smi as a fallback).  Reported as the recipe's clocks line."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (t, sm_mhz, max_mhz, reasons_bitmask)
        self.window = None  # (t0, t1) of the timed region
        self._stop = threading.Event()
        self._t = None
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _poll(self):
        if self.nvml is not None:
            p = self.nvml
            sm = p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM)
            reasons = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            return time.perf_counter(), float(sm), float(self.max_mhz), int(reasons)
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
        sm, mx = (float(v) for v in out.strip().split(","))
        return time.perf_counter(), sm, mx, 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._poll())
            except Exception:
                pass
            self._stop.wait(0.002 if self.nvml is not None else 0.2)

    def __enter__(self):
        try:
            self.samples.append(self._poll())
        except Exception:
            pass
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def summary(self):
        """Samples taken inside the timed window (the sampler runs from the warm-up on, so a
        short window is padded with the samples nearest to it until there are >= 5)."""
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sel = list(self.samples)
        if self.window is not None:
            t0, t1 = self.window
            inside = [x for x in self.samples if t0 <= x[0] <= t1]
            if len(inside) < 5:
                mid = 0.5 * (t0 + t1)
                inside = sorted(self.samples, key=lambda x: abs(x[0] - mid))[:5]
            sel = inside
        sm = [x[1] for x in sel]
        reasons = set()
        if self.nvml is not None:
            for name, const in self.REASONS:
                bit = getattr(self.nvml, const, 0)
                if any(x[3] & bit for x in sel):
                    reasons.add(name)
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(x[2] for x in sel),
               "reasons": sorted(reasons), "samples": len(sel),
               "source": "nvml" if self.nvml is not None else "nvidia-smi"}
        if self.window is not None:
            out["window_ms"] = round(1e3 * (self.window[1] - self.window[0]), 3)
        return out


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _timed_cpu(fn, items, budget_s, threads, min_items=1):
    """Run fn(item) over items until the budget is spent (>= min_items); (rate, done, seconds)."""
    from threadpoolctl import threadpool_limits

    with threadpool_limits(threads):
        fn(items[0])  # warm (page-in, BLAS threads)
        done, t0 = 0, time.perf_counter()
        for it in items:
            fn(it)
            done += 1
            if done >= min_items and time.perf_counter() - t0 >= budget_s:
                break
        el = time.perf_counter() - t0
    return done / el, done, el


def cpu_baseline(name, fn, items, unit_per_item, budget_s, sample_desc):
    """The oracle port (the reference's algorithm, NumPy/OpenBLAS fp64) on the host cores, all
    threads and threadpool_limits(1) (the reference harness's timing contract, harness.py:309)."""
    cores = len(os.sched_getaffinity(0))
    r_all, n_all, el_all = _timed_cpu(fn, items, budget_s, cores)
    r_one, n_one, el_one = _timed_cpu(fn, items, budget_s / 2, 1)
    return {"value": r_all * unit_per_item, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{sample_desc}: {n_all} in {el_all:.1f} s on {cores} threads; {n_one} in {el_one:.1f} s "
                      f"single-threaded ({name})",
            "single_thread": {"value": r_one * unit_per_item, "unit": UNIT, "cores": 1},
            "cpu_model": cpu_model()}


def cpu_oracle_rate(X, Q, h, budget_s=12.0, max_q=1024, threads=None, data=None):
    """NumPy oracle (the reference's algorithm) on a bounded query sample: queries/s."""
    from oracle import deann_oracle as O
    from threadpoolctl import threadpool_limits

    data = data if data is not None else O.Data(X)
    cores = threads or len(os.sched_getaffinity(0))
    with threadpool_limits(cores):
        O.naive_kde(data, "gaussian", h, Q[:2])  # warm
        done, t0 = 0, time.perf_counter()
        while done < max_q and (time.perf_counter() - t0) < budget_s:
            blk = Q[done: done + 16]
            if len(blk) == 0:
                break
            O.naive_kde(data, "gaussian", h, blk)
            done += len(blk)
        el = time.perf_counter() - t0
    return done / el, cores, done, el, data


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    import workloads
    from oracle import deann_oracle as O

    WL = WORKLOADS[args.workload]
    W = workloads.make(args.workload)
    h = _bandwidth_cpu_free(W)
    data = O.Data(W.X)
    cores = len(os.sched_getaffinity(0))
    # size each step so the whole run stays within ~2-3 minutes
    t0 = time.perf_counter()
    O.naive_kde(data, "gaussian", h, W.Q[:8])
    rate = 8 / max(time.perf_counter() - t0, 1e-6)
    per_step = int(max(4, min(256, rate * 120.0 / max(1, args.steps + args.warmup))))
    rng = np.random.default_rng(7)
    for _ in range(args.warmup):
        O.naive_kde(data, "gaussian", h, W.Q[rng.integers(0, len(W.Q), per_step)])
    times = []
    for _ in range(args.steps):
        sel = W.Q[rng.integers(0, len(W.Q), per_step)]
        t0 = time.perf_counter()
        O.naive_kde(data, "gaussian", h, sel)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": WL["metric"], "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WL["desc"], "bandwidth": h, "sample_queries_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"{per_step} random queries of the {len(W.Q):,} per step, full n={W.X.shape[0]:,} rows, "
                                   "oracle/deann_oracle.naive_kde (NumPy/OpenBLAS fp64, all host threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_H_CACHE = os.path.join(HERE, "tests", "golden", "bandwidths.json")


def _bandwidth_cpu_free(W):
    """Bandwidth of the workload from the committed manifest (written by the GPU fit)."""
    if os.path.exists(_H_CACHE):
        with open(_H_CACHE) as f:
            man = json.load(f)
        if W.name in man:
            return float(man[W.name]["h"])
    raise RuntimeError(f"no bandwidth for {W.name} in {_H_CACHE}; run bench.py --fit-bandwidth on a GPU first")


class Timer:
    """CUDA events on the launch stream around K steps, a barrier + synchronize on both sides,
    max over ranks; clocks sampled during the window."""

    def __init__(self, torch, dist, local):
        self.torch, self.dist, self.local = torch, dist, local

    def run(self, step, steps, warmup, clocks=None):
        torch = self.torch
        for i in range(warmup):
            step(i)
        torch.cuda.synchronize()
        if self.dist:
            self.dist.barrier()
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for i in range(steps):
            step(warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if clocks is not None:
            clocks.mark(t0, t1)
        ms = e0.elapsed_time(e1) / steps
        return self.max_over_ranks(ms)

    def wall(self, step, steps, warmup):
        """Host wall clock per step (e2e: host buffers, copies inside), max over ranks."""
        for i in range(warmup):
            step(i)
        self.torch.cuda.synchronize()
        if self.dist:
            self.dist.barrier()
        t0 = time.perf_counter()
        for i in range(steps):
            step(warmup + i)
        self.torch.cuda.synchronize()
        return self.max_over_ranks(1e3 * (time.perf_counter() - t0) / steps)

    def max_over_ranks(self, v):
        if not self.dist:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=f"cuda:{self.local}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t[0])


def _kernel_ms(lib, ds):
    import ctypes

    from paper_2107_02736_b200 import _lib

    kms, kfl, kby = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.dk_last_kernel_ms(ds.handle, ctypes.byref(kms), ctypes.byref(kfl), ctypes.byref(kby)))
    return kms.value, kfl.value, kby.value


def _launches(lib, ds):
    import ctypes

    from paper_2107_02736_b200 import _lib

    cnt = ctypes.c_int64()
    _lib.check(lib.dk_last_launch_count(ds.handle, ctypes.byref(cnt)))
    return int(cnt.value)


_SFU_MEASURED = {}


def _sfu_peak(peaks):
    """ex2/s of the SFU: measured on this GPU by dk_mufu_probe when available (the
    nominal 148 SMs x 16 / clk x max clock otherwise)."""
    return _SFU_MEASURED.get("value", 148 * 16 * peaks["sm_max_mhz"] * 1e6)


def _measure_sfu(local):
    import ctypes

    from paper_2107_02736_b200 import _lib

    v = ctypes.c_double()
    best = 0.0
    for _ in range(3):
        _lib.check(_lib.load().dk_mufu_probe(local, ctypes.byref(v)))
        best = max(best, v.value)
    _SFU_MEASURED["value"] = best


def run_ours(args):
    import torch

    import paper_2107_02736_b200 as g
    import workloads
    from paper_2107_02736_b200 import _lib

    ws, rank, local = _dist_env()
    if args.gpus > 1 and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    timer = Timer(torch, dist, local)
    _measure_sfu(local)
    WL = WORKLOADS[args.workload]
    W = workloads.make(args.workload)
    n, d = W.X.shape
    nq = W.Q.shape[0]
    lo, hi = (rank * n) // ws, ((rank + 1) * n) // ws
    t_fit = time.perf_counter()
    ds = g.Dataset.from_array(W.X[lo:hi], device=local, global_offset=lo, global_n=n)
    t_fit = time.perf_counter() - t_fit
    if ws == 1 and args.workload == "c2":
        h = g.fit_bandwidth(ds, W.pilot, "gaussian", 1e-3)
    else:
        h = _bandwidth_cpu_free(W)
    spec = g.KernelSpec("gaussian", h)
    stream = torch.cuda.current_stream()
    Qd = torch.from_numpy(W.Q).to(f"cuda:{local}")
    out = torch.empty(nq, dtype=torch.float64, device=f"cuda:{local}")
    lib = _lib.load()

    def step(_i):
        # each shard writes its contribution to the global mean (sum / global n): the all-reduce
        # (sum) of the shards is the KDE
        g.naive_kde_into(ds, spec, Qd, out, stream=stream.cuda_stream)
        if ws > 1:
            dist.all_reduce(out)

    with ClockSampler(local) as clocks:  # running from the warm-up on: the timed region is short
        for i in range(args.warmup):
            step(i)
        _lib.check(lib.dk_set_profiling(ds.handle, 1))
        ms = timer.run(step, args.steps, 0, clocks)
    launches = _launches(lib, ds) * args.steps
    kmsv = timer.max_over_ranks(_kernel_ms(lib, ds)[0])
    _lib.check(lib.dk_set_profiling(ds.handle, 0))
    # ---- e2e through the public API with pinned host buffers
    Qh = torch.from_numpy(W.Q).pin_memory().numpy()

    def e2e_step(_i):
        if ws == 1:
            return g.naive_kde(ds, spec, Qh).values
        tmp = torch.empty(nq, dtype=torch.float64, device=f"cuda:{local}")
        g.naive_kde_into(ds, spec, Qh, tmp, stream=stream.cuda_stream)
        dist.all_reduce(tmp)
        return tmp.cpu().numpy()

    with ClockSampler(local) as clk_e2e:
        e2e_ms = timer.wall(e2e_step, args.steps, max(10, args.warmup))
    # sustained: the same step repeated for ~2 s after the timed region (and the e2e steps, which
    # run first so they see the same board state as the timed region), so the board reaches its
    # steady power / clock state (a K-step window of a few ms may not); reported, not the value
    n_sus = max(args.steps, int(2000.0 / max(ms, 1e-3)))
    with ClockSampler(local) as clk_sus:
        ms_sus = timer.run(step, n_sus, 0, clk_sus)
    peaks = _peaks()
    n_local = hi - lo
    flops = 2.0 * d * nq * n_local
    ex2 = float(nq) * n_local
    tc_peak = peaks["bf16_tflops"] * 1e12
    sfu_peak = _sfu_peak(peaks)
    t_k = kmsv / 1e3
    t_bound = max(flops / tc_peak, ex2 / sfu_peak)
    traffic = None
    tpath = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(WL["traffic"] or "", {}).get("dram_bytes_per_launch")
    line = {
        "metric": WL["metric"], "value": nq / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": WL["dtype"], "data": "synthetic",
        "config": {"workload": WL["desc"], "bandwidth": h,
                   "parallelism": f"dataset-sharded x{ws}" if ws > 1 else "1 GPU",
                   "l2": WL["l2"], "fit_seconds": t_fit},
        "roofline": {
            "bound": "tensor", "achieved": flops / t_k / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
            "frac": (flops / t_k) / tc_peak, "traffic": traffic, "peak_source": peaks["source"],
            "kernel_ms": kmsv,
            "sfu": {"achieved": ex2 / t_k / 1e12, "peak": sfu_peak / 1e12, "unit": "Tex2/s",
                    "frac": (ex2 / t_k) / sfu_peak,
                    "peak_nominal": 148 * 16 * peaks["sm_max_mhz"] * 1e6 / 1e12,
                    "peak_note": "measured: dk_mufu_probe (ex2.approx.ftz.f32, 8 independent chains per thread, "
                                 "64 warps per SM, best of 3) on this GPU; nominal = 148 SMs x 16/clk x max clock"},
            "binding": "sfu" if ex2 / sfu_peak >= flops / tc_peak else "tensor",
            "frac_of_binding": t_bound / t_k,
        },
        "e2e": {"value": nq / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(nq * d * 8),
                "d2h_bytes_per_step": int(nq * 8), "api": "naive_kde(ds, KernelSpec, pinned host queries)",
                "clocks": clk_e2e.summary()},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "sustained": {"value": nq / (ms_sus / 1e3), "ms_per_step": ms_sus, "steps": n_sus,
                      "clocks": clk_sus.summary(),
                      "note": "the headline step repeated for ~2 s right after the timed region"},
    }
    if ws == 1 and not args.no_cpu_baseline:
        from oracle import deann_oracle as O

        odata = O.Data(W.X)
        line["cpu_baseline"] = cpu_baseline(
            "oracle/deann_oracle.naive_kde", lambda blk: O.naive_kde(odata, "gaussian", h, blk),
            [W.Q[i:i + 8] for i in range(0, 1024, 8)], 8, 10.0,
            f"blocks of 8 of the first 1,024 of the {nq:,} queries over all n={n:,} rows")
        # parity of the timed device output against the oracle on a query sample
        ref = O.naive_kde(odata, "gaussian", h, W.Q[:16])
        got = out[:16].cpu().numpy()
        line["parity_max_rel"] = float(np.max(np.abs(got - ref) / ref))
        del odata
    ds.free()
    del W
    if ws == 1 and not args.no_secondary:
        line["deann"], line["c3_exact"] = measure_deann_c3(args, local, timer)
    if not args.no_c5:
        c5 = measure_c5(args, ws, rank, local, dist, timer)
        if rank == 0:
            line["c5"] = c5
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _deann_oracle_fn(od, family, h, k, m):
    """The reference's DEANN with its BruteForceIndex (estimators.py:306-379, ann.py:105-121) and
    a numpy PCG64 Generator, per query."""
    from oracle import deann_oracle as O

    def fn(item):
        j, q = item
        O.deann(od, family, h, lambda y, kk: O.brute_force_knn(od, y, kk), q, k, m, rng=np.random.default_rng(j))

    return fn


def _deann_parity(od, family, h, k, m, Q, vals, seed, base, sel):
    """max relative error of GPU DEANN values against the oracle replaying the GPU's neighbours
    and Philox stream; plus whether the neighbour sets matched the brute force."""
    from oracle import deann_oracle as O
    from oracle.philox import IndexReplay, NeighborReplay

    err = 0.0
    for j in sel:
        ri, rd = O.brute_force_knn(od, Q[j], k)
        ref = O.deann(od, family, h, NeighborReplay(ri, rd), Q[j], k, m, rng=IndexReplay(seed, base + j, od.n))[0]
        err = max(err, abs(vals[j] - ref) / ref)
    return err


def measure_deann_c3(args, local, timer):
    """DEANN on config 3 (exact k=100 NN + m=1000 Philox samples): device value, e2e through
    deann_batch, per-kernel rooflines, clocks, parity, CPU baseline."""
    import torch

    import paper_2107_02736_b200 as g
    import workloads
    from oracle import deann_oracle as O
    from paper_2107_02736_b200 import _lib

    W = workloads.make("c3")
    h = _bandwidth_cpu_free(W)
    n, d = W.X.shape
    nq = W.Q.shape[0]
    ds = g.Dataset.from_array(W.X, device=local)
    spec = g.KernelSpec("gaussian", h)
    Qd = torch.from_numpy(W.Q).to(f"cuda:{local}")
    out = torch.empty(nq, dtype=torch.float64, device=f"cuda:{local}")
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    seed0 = 1234

    def step(i):
        _lib.check(lib.dk_deann(ds.handle, Qd.data_ptr(), nq, _lib.DK_GAUSSIAN, h, W.k, W.m, seed0 + i, 0,
                                out.data_ptr(), None, None, None, stream.cuda_stream))

    steps, warm = max(3, min(args.steps, 20)), max(3, args.warmup)
    exact = measure_c3_exact(args, local, timer, W, ds, spec, h, Qd, steps, warm)
    with ClockSampler(local) as clocks:
        ms = timer.run(step, steps, warm, clocks)
    launches = _launches(lib, ds)
    last_seed = seed0 + warm + steps - 1
    vals = out.cpu().numpy()  # the timed output (last step), before the profiling steps overwrite it
    # e2e: the public deann_batch with the GPU brute-force index, pinned host queries in, a
    # list of Estimates out (the values come back to the host inside every step)
    Qh = torch.from_numpy(W.Q).pin_memory().numpy()
    bf = g.BruteForceIndex(ds)

    def e2e_step(i):
        est = g.deann_batch(ds, spec, bf, Qh, W.k, W.m, rng=g.PhiloxSampler(seed0 + i))
        return est.values

    with ClockSampler(local) as clk_e2e:
        e2e_ms = timer.wall(e2e_step, max(steps, 20), 10)  # the first ~20 host-buffer calls run slower
    # per-kernel rooflines (library CUDA events on the launch stream, separate untimed steps):
    # the k-NN FILTER sweep against the tensor peak (2 d flops per (query, row) pair of the tiles
    # it visits — the ball-pruned lists) and the Philox gather against HBM (m accepted fp32 rows
    # of d floats per query)
    peaks = _peaks()
    kroof = {}
    for mode, name in ((1, "knn_filter_sweep"), (2, "sampling_gather")):
        _lib.check(lib.dk_set_profiling(ds.handle, mode))
        step(10_000 + mode)
        kms, kfl, kby = _kernel_ms(lib, ds)
        _lib.check(lib.dk_set_profiling(ds.handle, 0))
        if mode == 1:
            ach = kfl / (kms / 1e3) / 1e12
            dense = 2.0 * d * nq * n / (kms / 1e3) / 1e12
            kroof[name] = {"bound": "tensor", "achieved": ach, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                           "frac": ach / peaks["bf16_tflops"], "kernel_ms": kms, "dense_equivalent_tflops": dense}
        else:
            ach = kby / (kms / 1e3) / 1e9
            kroof[name] = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                           "frac": ach / peaks["hbm_gbs"], "kernel_ms": kms}
    res = {"metric": "DEANN queries/sec (exact k=100 NN + m=1000 Philox samples, gaussian) at n=1.2M, d=100",
           "value": nq / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warm,
           "higher_is_better": True, "gpu_launches": launches * steps,
           "e2e": {"value": nq / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(nq * d * 8),
                   "d2h_bytes_per_step": int(nq * 8),
                   "api": "deann_batch(ds, KernelSpec, BruteForceIndex(ds), pinned host queries, 100, 1000, "
                          "rng=PhiloxSampler) -> list[Estimate]", "clocks": clk_e2e.summary()},
           "kernel_rooflines": kroof, "clocks": clocks.summary(),
           "config": {"workload": "c3: 1,200,000 x 100 L2-normalised rows, 10,000 queries, h by median-1e-3 rule",
                      "bandwidth": h, "k": W.k, "m": W.m, "l2": "inputs larger than L2 (480 MB rows)"}}
    split3_only(timer, exact)
    ds.free()
    if not args.no_cpu_baseline:
        od = O.Data(W.X)
        sel = list(np.random.default_rng(3).choice(nq, 16, replace=False))
        res["parity_max_rel"] = _deann_parity(od, "gaussian", h, W.k, W.m, W.Q, vals, last_seed, 0, sel)
        res["parity_note"] = ("timed output (last step, seed %d) vs the oracle deann replaying the GPU's neighbours "
                              "and Philox stream, 16 seeded queries; gate 1e-5" % last_seed)
        res["cpu_baseline"] = cpu_baseline(
            "oracle deann + brute_force_knn, numpy PCG64", _deann_oracle_fn(od, "gaussian", h, W.k, W.m),
            [(j, W.Q[j]) for j in range(256)], 1, 10.0, f"the first 256 of the {nq:,} queries")
        ref = O.naive_kde(od, "gaussian", h, W.Q[exact.pop("_parity_sel")])
        exact["parity_max_rel"] = float(np.max(np.abs(exact.pop("_parity_vals") - ref) / ref))
        exact["cpu_baseline"] = cpu_baseline(
            "oracle/deann_oracle.naive_kde", lambda blk: O.naive_kde(od, "gaussian", h, blk),
            [W.Q[i:i + 8] for i in range(0, 512, 8)], 8, 6.0,
            f"blocks of 8 of the first 512 of the {nq:,} queries over all n={n:,} rows")
    exact.pop("_parity_sel", None)
    exact.pop("_parity_vals", None)
    exact.pop("_step", None)
    return res, exact


def measure_c3_exact(args, local, timer, W, ds, spec, h, Qd, steps, warm):
    """Exact KDE on config 3 (non-integer rows): the two-precision path (capi.cu kde_hybrid) —
    single-pass fp16 sweep of every pair, split3 sweep of the hot (block, tile) pairs, per-query
    bound — against the 1x roofline, with the split3-only time beside it."""
    import ctypes

    import torch

    import paper_2107_02736_b200 as g
    from paper_2107_02736_b200 import _lib

    lib = _lib.load()
    n, d = W.X.shape
    nq = W.Q.shape[0]
    stream = torch.cuda.current_stream()
    out = torch.empty(nq, dtype=torch.float64, device=f"cuda:{local}")

    def step(_i):
        g.naive_kde_into(ds, spec, Qd, out, stream=stream.cuda_stream)

    def stats():
        v = [ctypes.c_int64() for _ in range(4)]
        _lib.check(lib.dk_kde_stats(ds.handle, *[ctypes.byref(x) for x in v]))
        return [x.value for x in v]

    q0, f0, _, _ = stats()
    with ClockSampler(local) as clocks:
        for i in range(warm):
            step(i)
        q1, f1, _, _ = stats()
        _lib.check(lib.dk_set_profiling(ds.handle, 1))
        ms = timer.run(step, steps, 0, clocks)
    kms = _kernel_ms(lib, ds)[0]  # the single-pass fp16 sweep (every pair)
    _lib.check(lib.dk_set_profiling(ds.handle, 0))
    launches = _launches(lib, ds)
    q2, f2, hot, tot = stats()
    vals = out.cpu().numpy()
    Qh = torch.from_numpy(W.Q).pin_memory().numpy()
    with ClockSampler(local) as clk_e2e:  # right after the timed steps: the same board state
        e2e_ms = timer.wall(lambda i: g.naive_kde(ds, spec, Qh).values, steps, 5)
    peaks = _peaks()
    flops, ex2 = 2.0 * d * nq * n, float(nq) * n
    t_bound = max(flops / (peaks["bf16_tflops"] * 1e12), ex2 / _sfu_peak(peaks))
    sel = list(np.random.default_rng(5).choice(nq, 16, replace=False))
    return {
        "metric": "KDE queries/sec (exact naive KDE, gaussian) at n=1.2M, d=100",
        "value": nq / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warm,
        "higher_is_better": True, "gpu_launches": launches * steps,
        "dtype": "fp16 single pass for every pair + fp16 split3 for the hot tile halves (fp32 accumulate, "
                 "fp64 row sums), per-query a-posteriori bound of the fp16 part <= 2e-6",
        "two_precision": {"queries_served": q2 - q1, "fallback_queries": f2 - f1, "hot_block_tile_pairs": hot,
                          "block_tile_pairs": tot, "hot_fraction": hot / tot if tot > 0 else None,
                          "warmup_calls_served": q1 - q0},
        "roofline": {"bound": "sfu (1x: one exp2 per pair) / tensor (1x: one fp16 MMA pass)",
                     "kernel_ms_fp16_sweep": kms, "frac_of_1x_binding": t_bound / (ms / 1e3),
                     "fp16_sweep_frac_of_1x_binding": t_bound / (kms / 1e3),
                     "t_bound_ms": t_bound * 1e3, "sfu_peak_tex2s": _sfu_peak(peaks) / 1e12,
                     "tensor_peak_tflops": peaks["bf16_tflops"]},
        "e2e": {"value": nq / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(nq * d * 8),
                "d2h_bytes_per_step": int(nq * 8), "api": "naive_kde(ds, KernelSpec, pinned host queries)",
                "clocks": clk_e2e.summary()},
        "clocks": clocks.summary(),
        "config": {"workload": "c3: 1,200,000 x 100 L2-normalised rows, 10,000 queries, h by median-1e-3 rule",
                   "bandwidth": h, "l2": "inputs larger than L2 (307 MB fp16 operand + 480 MB rows)"},
        "_parity_sel": sel, "_parity_vals": vals[sel], "_step": step,
    }


def split3_only(timer, exact):
    """The round-1 all-split3 time of the same c3 exact step (DK_KDE_HYBRID=0), measured last:
    it is the most power-hungry run of the bench."""
    step = exact.pop("_step")
    os.environ["DK_KDE_HYBRID"] = "0"
    try:
        ms = timer.run(step, 5, 2)
    finally:
        del os.environ["DK_KDE_HYBRID"]
    exact["split3_only"] = {"value": exact["value"] * exact["ms_per_step"] / ms, "ms_per_step": ms,
                            "note": "DK_KDE_HYBRID=0: every pair in split3 (round-1 path), measured after DEANN"}


def measure_c5(args, ws, rank, local, dist, timer):
    """Config 5 (n = 8M, d = 96, 100,000 queries): exact KDE and DEANN (k = 100, m = 2,000).
    N = 1: the fused single-GPU calls; N > 1: dataset-sharded (ShardedKDE over NCCL)."""
    import torch

    import paper_2107_02736_b200 as g
    import workloads
    from paper_2107_02736_b200 import _lib
    from paper_2107_02736_b200.sharded import GpuShardEngine, ShardedKDE, TorchComm, shard_bounds

    W = workloads.make("c5")
    h = _bandwidth_cpu_free(W)
    n, d = W.X.shape
    nq = W.Q.shape[0]
    lo, hi = shard_bounds(n, ws, rank)
    t0 = time.perf_counter()
    ds = g.Dataset.from_array(W.X[lo:hi], device=local, global_offset=lo, global_n=n)
    fit_s = time.perf_counter() - t0
    spec = g.KernelSpec("gaussian", h)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    Qd = torch.from_numpy(W.Q).to(f"cuda:{local}")
    out = torch.empty(nq, dtype=torch.float64, device=f"cuda:{local}")
    sk = ShardedKDE(GpuShardEngine(None, global_offset=lo, global_n=n, device=local, dataset=ds), TorchComm()) \
        if ws > 1 else None
    seed0 = 777
    steps, warm = max(2, min(args.steps, 5)), max(3, min(args.warmup, 3))

    def exact_step(_i):
        g.naive_kde_into(ds, spec, Qd, out, stream=stream.cuda_stream)
        if ws > 1:
            dist.all_reduce(out)

    def deann_step(i):
        if ws == 1:
            _lib.check(lib.dk_deann(ds.handle, Qd.data_ptr(), nq, _lib.DK_GAUSSIAN, h, W.k, W.m, seed0 + i, 0,
                                    out.data_ptr(), None, None, None, stream.cuda_stream))
        else:
            out.copy_(sk.deann(None, spec, W.k, W.m, seed=seed0 + i, Qd=Qd))

    peaks = _peaks()
    with ClockSampler(local) as clk_exact:
        for i in range(warm):
            exact_step(i)
        _lib.check(lib.dk_set_profiling(ds.handle, 1))
        ms_exact = timer.run(exact_step, steps, 0, clk_exact)
    kms = timer.max_over_ranks(_kernel_ms(lib, ds)[0])
    _lib.check(lib.dk_set_profiling(ds.handle, 0))
    n_local = hi - lo
    flops, ex2 = 2.0 * d * nq * n_local, float(nq) * n_local
    t_bound = max(flops / (peaks["bf16_tflops"] * 1e12), ex2 / _sfu_peak(peaks))
    with ClockSampler(local) as clk_deann:
        ms_deann = timer.run(deann_step, steps, warm, clk_deann)
    res = {
        "config": {"workload": "c5: 8,000,000 x 96 mixture rows (Dirichlet weights), 100,000 queries, "
                               "h by median-1e-3 rule", "bandwidth": h, "k": W.k, "m": W.m,
                   "parallelism": f"dataset-sharded x{ws}" if ws > 1 else "1 GPU", "fit_seconds": fit_s,
                   "l2": "inputs larger than L2 (3.07 GB rows)"},
        "exact": {"metric": "KDE queries/sec (exact naive KDE, gaussian) at n=8M, d=96",
                  "value": nq / (ms_exact / 1e3), "unit": UNIT, "ms_per_step": ms_exact, "steps": steps,
                  "dtype": "fp16 split3 (fp32 accumulate, fp64 row sums)", "clocks": clk_exact.summary(),
                  "roofline": {"bound": "tensor x3 (split3) / sfu", "kernel_ms": kms,
                               "frac_of_1x_binding": t_bound / (kms / 1e3),
                               "achieved_tflops_algorithmic": flops / (kms / 1e3) / 1e12,
                               "achieved_tflops_issued_split3": 3 * flops / (kms / 1e3) / 1e12,
                               "peak_tflops": peaks["bf16_tflops"]}},
        "deann": {"metric": "DEANN queries/sec (exact k=100 NN + m=2000 Philox samples, gaussian) at n=8M, d=96",
                  "value": nq / (ms_deann / 1e3), "unit": UNIT, "ms_per_step": ms_deann, "steps": steps,
                  "clocks": clk_deann.summary()},
    }
    if ws == 1:
        Qh = torch.from_numpy(W.Q).pin_memory().numpy()
        e_ms = timer.wall(lambda i: g.naive_kde(ds, spec, Qh).values, 2, 1)
        res["exact"]["e2e"] = {"value": nq / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(nq * d * 8),
                               "d2h_bytes_per_step": int(nq * 8)}
        bf = g.BruteForceIndex(ds)
        d_ms = timer.wall(lambda i: g.deann_batch(ds, spec, bf, Qh, W.k, W.m, rng=g.PhiloxSampler(i)).values, 2, 1)
        res["deann"]["e2e"] = {"value": nq / (d_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(nq * d * 8),
                               "d2h_bytes_per_step": int(nq * 8)}
        deann_vals = out.cpu().numpy()
        last_seed = seed0 + warm + steps - 1
        ds.free()
        if not args.no_cpu_baseline:
            from oracle import deann_oracle as O

            naive_out = None
            od = O.Data(W.X)
            # parity: DEANN timed output (replay) and exact KDE on 4 queries over all 8M rows
            res["deann"]["parity_max_rel"] = _deann_parity(od, "gaussian", h, W.k, W.m, W.Q, deann_vals, last_seed,
                                                           0, [0, 50_000])
            ds2 = g.Dataset.from_array(W.X, device=local)
            naive_out = g.naive_kde(ds2, spec, W.Q[:4]).values
            ds2.free()
            ref = O.naive_kde(od, "gaussian", h, W.Q[:4])
            res["exact"]["parity_max_rel"] = float(np.max(np.abs(naive_out - ref) / ref))
            res["exact"]["cpu_baseline"] = cpu_baseline(
                "oracle/deann_oracle.naive_kde", lambda q: O.naive_kde(od, "gaussian", h, q.reshape(1, -1)),
                list(W.Q[:64]), 1, 8.0, "single queries of the first 64 over all 8M rows")
            res["deann"]["cpu_baseline"] = cpu_baseline(
                "oracle deann + brute_force_knn, numpy PCG64", _deann_oracle_fn(od, "gaussian", h, W.k, W.m),
                [(j, W.Q[j]) for j in range(64)], 1, 8.0, "the first 64 queries over all 8M rows")
            del od
    else:
        ds.free()
    return res


def fit_manifest():
    """Fit the median-1e-3 bandwidths of c2-c5 on the GPU and write tests/golden/bandwidths.json."""
    import paper_2107_02736_b200 as g
    import workloads

    man = {}
    if os.path.exists(_H_CACHE):
        with open(_H_CACHE) as f:
            man = json.load(f)
    for name, fams in [("c2", ["gaussian"]), ("c3", ["gaussian"]), ("c4", ["exponential", "laplacian"]),
                       ("c5", ["gaussian"])]:
        W = workloads.make(name)
        ds = g.Dataset.from_array(W.X)
        for fam in fams:
            t0 = time.perf_counter()
            h = g.fit_bandwidth(ds, W.pilot, fam, 1e-3)
            med = float(np.sort(g.naive_kde(ds, g.KernelSpec(fam, h), W.pilot).values)[(len(W.pilot) - 1) // 2])
            key = name if fam == W.family else f"{name}-{fam}"
            man[key] = {"family": fam, "h": h, "median_pilot_kde": med, "fit_seconds": time.perf_counter() - t0}
            print(key, man[key], flush=True)
        ds.free()
        del W
    with open(_H_CACHE, "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)


def _self_launch(args):
    """`python bench.py --gpus N` without torchrun: re-exec under torch.distributed.run with N
    ranks on this node (127.0.0.1 rendezvous); NCCL's init lines go to stderr."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execve(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2",
                    help="c2 (default; BASELINE configs[1], the metric's config) or c5 (scale-out config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the c3 DEANN object")
    ap.add_argument("--no-c5", action="store_true", help="skip the c5 (n = 8M) object")
    ap.add_argument("--fit-bandwidth", action="store_true", help="(re)write tests/golden/bandwidths.json")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.fit_bandwidth:
        fit_manifest()
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _self_launch(args)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init lines (comm size) to stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
