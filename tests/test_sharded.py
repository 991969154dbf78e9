"""Dataset-sharded orchestration (paper_2107_02736_b200.sharded) on CPU with gloo, world_size 2.

The per-shard arithmetic is the NumPy oracle (a test engine with the same
interface as GpuShardEngine); the code under test is the sharding, the
global row ids, the collectives and the DEANN combination.  Results must equal
the single-process oracle on the whole dataset.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import deann_oracle as O
from oracle.philox import IndexReplay, NeighborReplay, draws
from paper_2107_02736_b200.kernels import KernelSpec
from paper_2107_02736_b200.sharded import LocalComm, QueryShardedKDE, ShardedKDE, TorchComm, shard_bounds


def _fh(kernel):
    return kernel.family.value, kernel.bandwidth


class OracleShardEngine:
    """CPU stand-in for GpuShardEngine: one shard of a global dataset, oracle arithmetic."""

    def __init__(self, rows, *, global_offset, global_n):
        self.data = O.Data(rows)
        self.global_offset = int(global_offset)
        self.global_n = int(global_n)
        self.n_local = self.data.n
        self.d = self.data.d

    def queries(self, Q):
        return torch.as_tensor(np.ascontiguousarray(Q, dtype=np.float64))

    def kde_sums(self, Qd, kernel):
        fam, h = _fh(kernel)
        return torch.as_tensor(O.naive_kde(self.data, fam, h, Qd.numpy()) * self.n_local)

    def knn(self, Qd, k):
        nq = Qd.shape[0]
        kk = min(k, self.n_local)
        idx = np.full((nq, k), -1, dtype=np.int64)
        d2 = np.full((nq, k), np.inf)
        for j, q in enumerate(Qd.numpy()):
            i, dd = O.brute_force_knn(self.data, q, kk)
            idx[j, :kk] = i + self.global_offset
            d2[j, :kk] = dd
        return torch.as_tensor(idx), torch.as_tensor(d2)

    def merge_topk(self, ig, dg, k):
        ig, dg = ig.numpy(), dg.numpy()
        nq = ig.shape[1]
        idx = np.empty((nq, k), dtype=np.int64)
        d2 = np.empty((nq, k))
        for j in range(nq):
            ii, dd = ig[:, j, :].ravel(), dg[:, j, :].ravel()
            keep = ii >= 0
            ii, dd = ii[keep], dd[keep]
            order = np.lexsort((ii, dd))[:k]
            idx[j], d2[j] = ii[order], dd[order]
        return torch.as_tensor(idx), torch.as_tensor(d2)

    def sample_sums(self, Qd, kernel, m, seed, query_base, excl, export=None):
        fam, h = _fh(kernel)
        out = np.zeros(Qd.shape[0])
        for j, q in enumerate(Qd.numpy()):
            stream = draws(seed, query_base + j, 0, 20 * m + 1000, self.global_n)
            if excl is not None:
                stream = stream[~np.isin(stream, excl[j].numpy())]
            acc = stream[:m]
            if export is not None:
                export[j] = torch.as_tensor(acc)
            loc = acc - self.global_offset
            loc = loc[(loc >= 0) & (loc < self.n_local)]
            out[j] = O.kernel_rows(self.data.x64, self.data.sq_norms, fam, h, loc, q).sum()
        return torch.as_tensor(out)

    def row_sums(self, Qd, kernel, rows):
        fam, h = _fh(kernel)
        out = np.zeros(Qd.shape[0])
        for j, q in enumerate(Qd.numpy()):
            loc = rows[j].numpy() - self.global_offset
            loc = loc[(loc >= 0) & (loc < self.n_local)]
            out[j] = O.kernel_rows(self.data.x64, self.data.sq_norms, fam, h, loc, q).sum()
        return torch.as_tensor(out)

    def combine(self, kernel, k, m, nbr_d2, z1_l1_sum, z2_sum):
        """estimators.py:344-372: Z1 from the neighbour distances (L2) or the L1 sums, Z2 = sum / m."""
        fam, h = _fh(kernel)
        N = self.global_n
        t = nbr_d2 if nbr_d2 is not None else (z2_sum if z2_sum is not None else z1_l1_sum)
        val = np.zeros(t.shape[0])
        if k > 0:
            z1 = z1_l1_sum.numpy() / k if fam == "laplacian" else \
                O.kernel_from_sql2(fam, h, nbr_d2.numpy().copy()).mean(axis=1)
            val += (k / N) * z1
        if m > 0:
            val += ((N - k) / N) * (z2_sum.numpy() / m)
        return torch.as_tensor(val)


class OracleReplicaEngine:
    """CPU stand-in for GpuReplicaEngine (query-sharded mode): the whole dataset, oracle arithmetic."""

    def __init__(self, rows):
        self.data = O.Data(rows)
        self.n = self.data.n
        self.d = self.data.d

    def queries(self, Q):
        return torch.as_tensor(np.ascontiguousarray(Q, dtype=np.float64))

    def naive(self, Qd, kernel):
        fam, h = _fh(kernel)
        return torch.as_tensor(O.naive_kde(self.data, fam, h, Qd.numpy()) if Qd.shape[0] else np.zeros(0))

    def knn(self, Qd, k):
        out = [O.brute_force_knn(self.data, q, k) for q in Qd.numpy()]
        idx = np.array([o[0] for o in out], dtype=np.int64).reshape(-1, k)
        d2 = np.array([o[1] for o in out]).reshape(-1, k)
        return torch.as_tensor(idx), torch.as_tensor(d2)

    def deann(self, Qd, kernel, k, m, seed, query_base, export_samples=None):
        fam, h = _fh(kernel)
        vals = np.zeros(Qd.shape[0])
        for j, q in enumerate(Qd.numpy()):
            i, dd = O.brute_force_knn(self.data, q, k) if k else (np.empty(0, np.int64), np.empty(0))
            vals[j] = O.deann(self.data, fam, h, NeighborReplay(i, dd), q, k, m,
                              rng=IndexReplay(seed, query_base + j, self.n))[0]
            if export_samples is not None:
                stream = draws(seed, query_base + j, 0, 20 * m + 1000, self.n)
                export_samples[j] = torch.as_tensor(stream[~np.isin(stream, i)][:m])
        return torch.as_tensor(vals)


def _problem():
    rng = np.random.default_rng(5)
    X = rng.normal(size=(601, 5)).astype(np.float32)
    Q = rng.normal(size=(7, 5))
    return X, Q


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Q = _problem()
        lo, hi = shard_bounds(X.shape[0], world, rank)
        sk = ShardedKDE(OracleShardEngine(X[lo:hi], global_offset=lo, global_n=X.shape[0]), TorchComm())
        out = {}
        for fam, h in [("gaussian", 1.2), ("exponential", 0.9), ("laplacian", 2.0)]:
            out[f"naive_{fam}"] = sk.naive_kde(Q, KernelSpec(fam, h)).numpy()
            out[f"deann_{fam}"] = sk.deann(Q, KernelSpec(fam, h), 12, 40, seed=99, query_base=3).numpy()
        idx, d2 = sk.knn(Q, 12)
        out["knn_idx"], out["knn_d2"] = idx.numpy(), d2.numpy()
        acc = torch.zeros((Q.shape[0], 40), dtype=torch.int64)
        out["ds_deann"] = sk.deann(Q, KernelSpec("gaussian", 1.2), 12, 40, seed=7, query_base=11,
                                   export_samples=acc).numpy()
        out["ds_acc"] = acc.numpy()
        # query-sharded mode: every rank holds all rows, evaluates its slice of the queries
        qs = QueryShardedKDE(OracleReplicaEngine(X), TorchComm(), rank, world)
        out["qs_naive"] = qs.naive_kde(Q, KernelSpec("gaussian", 1.2)).numpy()
        qi, qd = qs.knn(Q, 12)
        out["qs_knn_idx"], out["qs_knn_d2"] = qi.numpy(), qd.numpy()
        v, a = qs.deann(Q, KernelSpec("gaussian", 1.2), 12, 40, seed=7, query_base=11, export_samples=True)
        out["qs_deann"], out["qs_acc"] = v.numpy(), a.numpy()
        if rank == 0:
            results.update(out)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def sharded_results():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    return dict(results)


def test_sharded_naive_equals_whole(sharded_results):
    X, Q = _problem()
    d = O.Data(X)
    for fam, h in [("gaussian", 1.2), ("exponential", 0.9), ("laplacian", 2.0)]:
        np.testing.assert_allclose(sharded_results[f"naive_{fam}"], O.naive_kde(d, fam, h, Q), rtol=1e-12)


def test_sharded_knn_equals_whole(sharded_results):
    X, Q = _problem()
    d = O.Data(X)
    for j, q in enumerate(Q):
        i, dd = O.brute_force_knn(d, q, 12)
        np.testing.assert_array_equal(sharded_results["knn_idx"][j], i)
        np.testing.assert_allclose(sharded_results["knn_d2"][j], dd, rtol=1e-12)


def test_sharded_deann_equals_whole_with_replay(sharded_results):
    X, Q = _problem()
    d = O.Data(X)
    for fam, h in [("gaussian", 1.2), ("exponential", 0.9), ("laplacian", 2.0)]:
        for j, q in enumerate(Q):
            i, dd = O.brute_force_knn(d, q, 12)
            ref = O.deann(d, fam, h, NeighborReplay(i, dd), q, 12, 40, rng=IndexReplay(99, 3 + j, d.n))[0]
            assert sharded_results[f"deann_{fam}"][j] == pytest.approx(ref, rel=1e-12)


def test_query_sharded_equals_dataset_sharded(sharded_results):
    """SURVEY §7 test plan: both modes on the same seeds give identical k-NN sets and identical
    accepted sample ids; the values agree (here both are fp64 oracle arithmetic)."""
    r = sharded_results
    np.testing.assert_array_equal(r["qs_knn_idx"], r["knn_idx"])
    np.testing.assert_allclose(r["qs_knn_d2"], r["knn_d2"], rtol=1e-12)
    np.testing.assert_array_equal(r["qs_acc"], r["ds_acc"])
    np.testing.assert_allclose(r["qs_deann"], r["ds_deann"], rtol=1e-12)
    np.testing.assert_allclose(r["qs_naive"], r["naive_gaussian"], rtol=1e-12)


def test_local_comm_single_shard_matches():
    X, Q = _problem()
    sk = ShardedKDE(OracleShardEngine(X, global_offset=0, global_n=X.shape[0]), LocalComm())
    np.testing.assert_allclose(sk.naive_kde(Q, KernelSpec("gaussian", 1.2)).numpy(), O.naive_kde(O.Data(X), "gaussian", 1.2, Q),
                               rtol=1e-14)
    with pytest.raises(ValueError):
        sk.deann(Q, KernelSpec("gaussian", 1.0), X.shape[0], 5, seed=1)


def test_shard_bounds_partition():
    for n in (1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
