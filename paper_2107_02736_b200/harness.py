"""Batch-aware experiment runner — the GPU side of the reference's
``harness._Runner`` (harness.py:199-270) and of its timed repetition loop
(``_run_repetitions``, harness.py:344-381).

The reference times one ``_Runner.query(y)`` call per query, single-threaded: on the GPU
that is launch-bound.  ``BatchRunner`` keeps the same preprocessing split (index build and
permutation timed separately), the same ``reset(rep_seed)`` / ``warm`` / ``touch`` /
``query(y)`` protocol, and adds ``query_batch(Q)``: one device call for the whole
repetition whose estimates equal the per-query loop's, query for query (the uniform
sampler is a Philox stream per query position, the permuted sampler threads the shared
cursor in query order exactly as repeated ``rsp_kde`` / ``deann`` calls do).
``evaluate_batch`` is ``harness.evaluate`` with the batch timed instead of each query:
``mean_query_time_ms`` = batch time / queries.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .ann import BruteForceIndex, knn_batch
from .data import as_gpu_dataset
from .estimators import Estimate, EstimateList, RspState, deann, deann_batch, naive_kde, rs_kde, rsp_kde
from .ivf import IvfAnnIndex, ivf_build
from .kernels import as_spec
from .sampler import PhiloxSampler

__all__ = ["BatchRunner", "evaluate_batch", "relative_error", "ESTIMATORS", "DEFAULT_KDE_FLOOR"]

ESTIMATORS = ("naive", "rs", "rsp", "deann", "deannp")  # harness.py:53
DEFAULT_KDE_FLOOR = 1e-16                               # analysis.py:40
DEFAULT_REPETITIONS = 5                                 # harness.py:55


@dataclass
class ErrorReport:
    """analysis.py:83-88"""

    per_query_rel_err: np.ndarray
    mean_rel_err: float
    excluded_count: int


def relative_error(estimates, exact, floor: float = DEFAULT_KDE_FLOOR) -> ErrorReport:
    """|Z - mu| / mu over queries with mu >= floor (analysis.py:326-343)."""
    z = np.asarray(estimates, dtype=np.float64).ravel()
    mu = np.asarray(exact, dtype=np.float64).ravel()
    if z.shape != mu.shape:
        raise ValueError(f"length mismatch: {z.shape[0]} estimates vs {mu.shape[0]} exact values")
    inc = mu >= floor
    rel = np.abs(z[inc] - mu[inc]) / mu[inc]
    return ErrorReport(per_query_rel_err=rel, mean_rel_err=float(rel.mean()) if rel.size else float("nan"),
                       excluded_count=int((~inc).sum()))


class BatchRunner:
    """Per-configuration estimator with preprocessing split out (harness._Runner,
    harness.py:199-270), plus a whole-repetition ``query_batch``."""

    def __init__(self, estimator: str, train, kernel, params: dict, seed: int, index_cache: dict | None = None):
        if estimator not in ESTIMATORS:
            raise ValueError(f"unknown estimator {estimator!r}; choose from {ESTIMATORS}")
        self.estimator = estimator
        self.train = as_gpu_dataset(train)
        self.kernel = as_spec(kernel)
        self.params = params
        self.seed = seed
        self.rng = None
        self.state = None
        self.ann = None
        self.k = params.get("k")
        self.m = params.get("m")
        t0 = time.perf_counter()
        cached_build_s = 0.0
        if estimator in ("deann", "deannp") and self.k and self.k > 0:
            if "n_clusters" in params:
                key = (params["n_clusters"], seed)
                if index_cache is not None and key in index_cache:
                    index, cached_build_s = index_cache[key]
                else:
                    b0 = time.perf_counter()
                    index = ivf_build(self.train, params["n_clusters"], seed)
                    if index_cache is not None:
                        index_cache[key] = (index, time.perf_counter() - b0)
                self.ann = IvfAnnIndex(self.train, index, params["n_probe"])
            else:  # exact neighbours (the north star's brute-force index)
                self.ann = BruteForceIndex(self.train)
        if estimator in ("rsp", "deannp"):
            self.state = RspState.from_dataset(self.train, seed)
        self.preprocessing_s = (time.perf_counter() - t0) + cached_build_s

    def reset(self, rep_seed: int) -> None:
        if self.estimator in ("rs", "deann"):
            self.rng = PhiloxSampler(rep_seed)
        if self.estimator in ("rsp", "deannp"):
            self.state = RspState.from_dataset(self.train, rep_seed)

    def warm(self, queries) -> None:
        """One untimed pass over the first queries (harness.py:243-251), state re-seeded."""
        self.reset(self.seed)
        q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
        self.query_batch(q[: min(2, len(q))])
        self.reset(self.seed)

    def touch(self) -> None:
        """The reference pages in host copies here (harness.py:253-256); device state is resident."""

    def query(self, y) -> Estimate:
        """One query, exactly the reference's dispatch (harness.py:258-270)."""
        est = self.estimator
        if est == "naive":
            b = naive_kde(self.train, self.kernel, np.asarray(y, dtype=np.float64).reshape(1, -1))
            return Estimate(value=float(b.values[0]), kernel_evals=self.train.n, neighbors_used=0, samples_used=0)
        if est == "rs":
            return rs_kde(self.train, self.kernel, y, self.m, self.rng)
        if est == "rsp":
            return rsp_kde(self.state, self.kernel, y, self.m)
        if est == "deann":
            return deann(self.train, self.kernel, self.ann, y, self.k, self.m, rng=self.rng)
        return deann(self.train, self.kernel, self.ann, y, self.k, self.m, rsp_state=self.state)

    def query_batch(self, Q) -> list[Estimate]:
        """The whole batch in one device call; equals [query(y) for y in Q] in query order."""
        Q = np.atleast_2d(np.asarray(Q, dtype=np.float64))
        est, n = self.estimator, self.train.n
        if est == "naive":
            b = naive_kde(self.train, self.kernel, Q)
            return EstimateList(b.values, n, 0, 0)
        if est == "rs":  # rs_kde per query == deann(k=0) per query on the same sampler positions
            return deann_batch(self.train, self.kernel, None, Q, 0, self.m, rng=self.rng)
        if est == "rsp":
            return deann_batch(self.train, self.kernel, None, Q, 0, self.m, rsp_state=self.state)
        if est == "deann":
            return deann_batch(self.train, self.kernel, self.ann, Q, self.k or 0, self.m, rng=self.rng)
        return deann_batch(self.train, self.kernel, self.ann, Q, self.k or 0, self.m, rsp_state=self.state)


def _sync():
    try:
        import torch

        if torch.cuda.is_available():
            torch.cuda.synchronize()
    except ImportError:  # pragma: no cover
        pass


def evaluate_batch(estimator: str, train, kernel, test_queries, exact_values, params: dict, *, seed: int = 0,
                   repetitions: int = DEFAULT_REPETITIONS, kde_floor: float = DEFAULT_KDE_FLOOR,
                   timing: bool = True, compute_recall: bool = True):
    """``harness.evaluate`` (harness.py:450-473, :288-381) over batches: per repetition,
    reset(seed + rep) and one timed ``query_batch``; returns (row dict with the reference's
    ResultRow fields, per-query records)."""
    spec = as_spec(kernel)
    Q = np.atleast_2d(np.asarray(test_queries, dtype=np.float64))
    exact = np.asarray(exact_values, dtype=np.float64).ravel()
    if len(exact) != Q.shape[0]:
        raise ValueError("ground truth length does not match query count")
    runner = BatchRunner(estimator, train, spec, params, seed)
    if timing:
        w0 = time.perf_counter()
        runner.warm(Q)
        runner.preprocessing_s += time.perf_counter() - w0
    errs, excluded, times, evals, per_query = [], [], [], [], []
    for rep in range(repetitions):
        runner.reset(seed + rep)
        runner.touch()
        _sync()
        t0 = time.perf_counter()
        out = runner.query_batch(Q)
        vals = np.asarray(out.values if isinstance(out, EstimateList) else [e.value for e in out])
        _sync()
        dt = time.perf_counter() - t0
        ke = np.asarray(out.kernel_evals if isinstance(out, EstimateList) else [e.kernel_evals for e in out])
        times.append(dt / Q.shape[0])
        evals.extend(ke.tolist())
        rep_err = relative_error(vals, exact, floor=kde_floor)
        errs.append(rep_err.mean_rel_err)
        excluded.append(rep_err.excluded_count)
        for j in range(Q.shape[0]):
            per_query.append({"repetition": rep, "query_index": j, "estimate": float(vals[j]),
                              "exact": float(exact[j]),
                              "rel_err": abs(vals[j] - exact[j]) / exact[j] if exact[j] >= kde_floor else None,
                              "query_time_ms": dt / Q.shape[0] * 1e3 if timing else None,
                              "kernel_evals": int(ke[j])})
    recall = None
    if compute_recall and isinstance(runner.ann, IvfAnnIndex) and runner.k:
        k = min(runner.k, runner.train.n)
        ex_idx, _ = knn_batch(runner.train, Q, k)
        ap_idx, _, cnt = runner.ann.query_batch(Q, runner.k)
        recall = float(np.mean([np.intersect1d(ap_idx[j, :cnt[j]], ex_idx[j]).size / k for j in range(Q.shape[0])]))
    row = {"estimator": estimator, "k": params.get("k"), "m": params.get("m"),
           "n_clusters": params.get("n_clusters"), "n_probe": params.get("n_probe"), "bandwidth": spec.bandwidth,
           "mean_rel_err": float(np.mean(errs)), "mean_query_time_ms": 1e3 * float(np.mean(times)) if timing else None,
           "mean_kernel_evals": float(np.mean(evals)), "recall": recall, "repetitions": repetitions,
           "excluded_count": int(np.max(excluded)), "preprocessing_s": runner.preprocessing_s, "timed_out": False,
           "selected": False}
    return row, per_query

