"""Multi-GPU modes: dataset-sharded (X row-split) and query-sharded (X replicated).

One process per GPU (torch.distributed, backend "nccl"); rank r holds rows
[offset_r, offset_r + n_r) of the global dataset, fitted with dk_fit's
global_offset / global_n so every row id it reports is global.  Per query
batch:

* exact KDE  : each rank computes its partial kernel SUMS (dk_naive with
               DK_OUT_SUM) -> all_reduce(sum, fp64) -> / N.
* k-NN       : each rank its local exact top-k (dk_knn, global ids) ->
               all_gather -> deterministic (d2, idx) merge (dk_merge_topk) on
               every rank.
* DEANN      : global k-NN as above; Z1 from the merged exact distances (L2
               families) or an all_reduce of per-shard L1 kernel sums over the
               global neighbour ids (laplacian); Z2: every rank walks the SAME
               Philox stream over [0, N) with the same global exclusion list and
               sums the accepted samples that fall in its shard (dk_sample),
               all_reduce -> the single-GPU estimate up to fp64 summation order.
               value = (k/N) Z1 + ((N-k)/N) Z2   (estimators.py:372), combined on the
               device by dk_deann_combine (the same kernel as the single-GPU dk_deann).

Query-sharded mode (`QueryShardedKDE`): every rank fits the whole dataset, takes a
contiguous slice of the query batch and runs the fused single-GPU path on it (query
j keeps its global position, so its Philox stream — and every accepted sample id —
is the one the single-GPU and dataset-sharded runs draw); the slices are gathered.
No collective on the data path besides that final gather.

The per-shard arithmetic is an engine object; `GpuShardEngine` (the product)
drives the C-ABI, the collectives go through a `Comm`.  Tests substitute a
CPU engine built on the oracle and a gloo process group to cover the
orchestration without GPUs (tests/test_sharded.py).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .data import Dataset
from .kernels import as_spec

__all__ = ["GpuShardEngine", "GpuReplicaEngine", "TorchComm", "LocalComm", "ShardedKDE", "QueryShardedKDE",
           "shard_bounds"]


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of `rank` (sizes differ by at most one)."""
    return (rank * n) // world, ((rank + 1) * n) // world


class TorchComm:
    """Collectives over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather(self, t):
        import torch

        world = self.dist.get_world_size(self.group)
        out = [torch.empty_like(t) for _ in range(world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out)


class LocalComm:
    """Single process, several engines (e.g. shards on one GPU): collectives are local."""

    def all_reduce_sum(self, t):
        return t

    def all_gather(self, t):
        return t.unsqueeze(0)


class GpuShardEngine:
    """One shard on one GPU: fits rows [offset, offset+n) of a global dataset of N rows."""

    def __init__(self, rows, *, global_offset: int, global_n: int, device: int = 0, precision: str = "auto",
                 dataset: Dataset | None = None):
        import torch

        self.torch = torch
        self.device = torch.device("cuda", device)
        self.ds = dataset if dataset is not None else Dataset.from_array(
            rows, device=device, precision=precision, global_offset=global_offset, global_n=global_n)
        self.global_n = int(global_n)
        self.global_offset = int(global_offset)
        self.n_local = self.ds.n
        self.d = self.ds.d

    @classmethod
    def from_file(cls, path, world: int, rank: int, *, device: int = 0, precision: str = "auto"):
        """This rank's contiguous row shard of a DEANN1 file, streamed file -> device (row f4)."""
        from .data import file_info, load

        n, _ = file_info(path)
        lo, hi = shard_bounds(n, world, rank)
        ds = load(path, device=device, precision=precision, rows=(lo, hi - lo)) if hi - lo < n else \
            load(path, device=device, precision=precision)
        return cls(None, global_offset=lo, global_n=n, device=device, dataset=ds)

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def queries(self, Q):
        return self.torch.as_tensor(np.ascontiguousarray(Q, dtype=np.float64), device=self.device)

    def kde_sums(self, Qd, kernel):
        spec = as_spec(kernel)
        out = self.torch.empty(Qd.shape[0], dtype=self.torch.float64, device=self.device)
        _lib.check(_lib.load().dk_naive(self.ds.handle, Qd.data_ptr(), Qd.shape[0], _lib.family_code(spec.family),
                                        spec.bandwidth, _lib.DK_OUT_SUM, out.data_ptr(), self._stream()))
        return out

    def knn(self, Qd, k):
        kk = min(k, self.n_local)
        nq = Qd.shape[0]
        idx = self.torch.full((nq, k), -1, dtype=self.torch.int64, device=self.device)
        d2 = self.torch.full((nq, k), float("inf"), dtype=self.torch.float64, device=self.device)
        if kk < k:  # shard smaller than k: pad with (inf, -1)
            ti = self.torch.empty((nq, kk), dtype=self.torch.int64, device=self.device)
            td = self.torch.empty((nq, kk), dtype=self.torch.float64, device=self.device)
            _lib.check(_lib.load().dk_knn(self.ds.handle, Qd.data_ptr(), nq, kk, ti.data_ptr(), td.data_ptr(),
                                          self._stream()))
            idx[:, :kk] = ti
            d2[:, :kk] = td
        else:
            _lib.check(_lib.load().dk_knn(self.ds.handle, Qd.data_ptr(), nq, k, idx.data_ptr(), d2.data_ptr(),
                                          self._stream()))
        return idx, d2

    def merge_topk(self, idx_parts, d2_parts, k):
        parts, nq = idx_parts.shape[0], idx_parts.shape[1]
        idx = self.torch.empty((nq, k), dtype=self.torch.int64, device=self.device)
        d2 = self.torch.empty((nq, k), dtype=self.torch.float64, device=self.device)
        _lib.check(_lib.load().dk_merge_topk(parts, nq, k, idx_parts.contiguous().data_ptr(),
                                             d2_parts.contiguous().data_ptr(), idx.data_ptr(), d2.data_ptr(),
                                             self._stream()))
        return idx, d2

    def sample_sums(self, Qd, kernel, m, seed, query_base, excl, export=None):
        """Kernel sums of this shard's rows among the first m accepted draws of each query's
        global stream; `export` (nq, m) int64 device tensor receives the accepted ids."""
        spec = as_spec(kernel)
        nq = Qd.shape[0]
        z = self.torch.empty(nq, dtype=self.torch.float64, device=self.device)
        ex = excl.contiguous() if excl is not None else None
        _lib.check(_lib.load().dk_sample(self.ds.handle, Qd.data_ptr(), nq, _lib.family_code(spec.family),
                                         spec.bandwidth, m, seed, query_base,
                                         ex.data_ptr() if ex is not None else None, None,
                                         ex.shape[1] if ex is not None else 0, z.data_ptr(),
                                         export.data_ptr() if export is not None else None, None,
                                         self._stream()))
        return z

    def row_sums(self, Qd, kernel, rows):
        spec = as_spec(kernel)
        nq = Qd.shape[0]
        out = self.torch.empty(nq, dtype=self.torch.float64, device=self.device)
        r = rows.contiguous()
        _lib.check(_lib.load().dk_eval_rows(self.ds.handle, Qd.data_ptr(), nq, _lib.family_code(spec.family),
                                            spec.bandwidth, r.data_ptr(), None, r.shape[1], out.data_ptr(),
                                            self._stream()))
        return out

    def combine(self, kernel, k, m, nbr_d2, z1_l1_sum, z2_sum):
        """value = (k/N) Z1 + ((N-k)/N) Z2 on the device (dk_deann_combine, the single-GPU kernel)."""
        spec = as_spec(kernel)
        t = nbr_d2 if nbr_d2 is not None else (z2_sum if z2_sum is not None else z1_l1_sum)
        nq = t.shape[0]
        out = self.torch.empty(nq, dtype=self.torch.float64, device=self.device)
        ptr = lambda x: x.contiguous().data_ptr() if x is not None else None  # noqa: E731
        _lib.check(_lib.load().dk_deann_combine(nq, _lib.family_code(spec.family), spec.bandwidth, k, m,
                                                self.global_n, ptr(nbr_d2), ptr(z1_l1_sum), ptr(z2_sum),
                                                out.data_ptr(), self._stream()))
        return out


class ShardedKDE:
    """The reference's batch estimators over a row-sharded dataset (one engine per rank)."""

    def __init__(self, engine, comm):
        self.engine = engine
        self.comm = comm
        self.N = engine.global_n

    def naive_kde(self, Q, kernel):
        Qd = self.engine.queries(Q)
        s = self.comm.all_reduce_sum(self.engine.kde_sums(Qd, kernel))
        return s / float(self.N)

    def knn(self, Q, k, Qd=None):
        if not 1 <= k <= self.N:
            raise ValueError(f"k={k} out of range [1, {self.N}]")
        Qd = self.engine.queries(Q) if Qd is None else Qd
        idx, d2 = self.engine.knn(Qd, k)
        ig = self.comm.all_gather(idx)
        dg = self.comm.all_gather(d2)
        return self.engine.merge_topk(ig, dg, k)

    def deann(self, Q, kernel, k, m, *, seed: int, query_base: int = 0, Qd=None, export_samples=None):
        """Batch DEANN with exact global k-NN and the global Philox sampler.  `Qd`: queries already
        on the device (Q is then ignored); `export_samples`: (nq, m) int64 device tensor that
        receives the accepted sample ids (the same on every rank)."""
        spec = as_spec(kernel)
        N = self.N
        if not 0 <= k <= N:
            raise ValueError(f"k={k} out of range [0, {N}]")
        if m < 0:
            raise ValueError(f"m={m} must be >= 0")
        if m > 0 and k >= N:
            raise ValueError("m > 0 requires k + 1 <= n so the remainder is nonempty")
        Qd = self.engine.queries(Q) if Qd is None else Qd
        nq = Qd.shape[0]
        d2 = z1s = z2s = None
        excl = None
        if k > 0:
            idx, d2 = self.knn(None, k, Qd=Qd)
            excl = idx
            if spec.family.value == "laplacian":
                z1s = self.comm.all_reduce_sum(self.engine.row_sums(Qd, spec, idx))
        if m > 0:
            z2s = self.comm.all_reduce_sum(self.engine.sample_sums(Qd, spec, m, seed, query_base, excl,
                                                                   export=export_samples))
        if k == 0 and m == 0:
            return Qd.new_zeros(nq)
        return self.engine.combine(spec, k, m, d2, z1s, z2s)


class GpuReplicaEngine:
    """The whole dataset on this rank's GPU (query-sharded mode): fused single-GPU calls."""

    def __init__(self, X=None, *, device: int = 0, precision: str = "auto", dataset: Dataset | None = None):
        import torch

        self.torch = torch
        self.device = torch.device("cuda", device)
        self.ds = dataset if dataset is not None else Dataset.from_array(X, device=device, precision=precision)
        self.n = self.ds.n
        self.d = self.ds.d

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def queries(self, Q):
        return self.torch.as_tensor(np.ascontiguousarray(Q, dtype=np.float64), device=self.device)

    def naive(self, Qd, kernel):
        spec = as_spec(kernel)
        out = self.torch.empty(Qd.shape[0], dtype=self.torch.float64, device=self.device)
        if Qd.shape[0]:
            _lib.check(_lib.load().dk_naive(self.ds.handle, Qd.data_ptr(), Qd.shape[0], _lib.family_code(spec.family),
                                            spec.bandwidth, 0, out.data_ptr(), self._stream()))
        return out

    def knn(self, Qd, k):
        nq = Qd.shape[0]
        idx = self.torch.empty((nq, k), dtype=self.torch.int64, device=self.device)
        d2 = self.torch.empty((nq, k), dtype=self.torch.float64, device=self.device)
        if nq:
            _lib.check(_lib.load().dk_knn(self.ds.handle, Qd.data_ptr(), nq, k, idx.data_ptr(), d2.data_ptr(),
                                          self._stream()))
        return idx, d2

    def deann(self, Qd, kernel, k, m, seed, query_base, export_samples=None):
        spec = as_spec(kernel)
        out = self.torch.empty(Qd.shape[0], dtype=self.torch.float64, device=self.device)
        if Qd.shape[0]:
            _lib.check(_lib.load().dk_deann(self.ds.handle, Qd.data_ptr(), Qd.shape[0], _lib.family_code(spec.family),
                                            spec.bandwidth, k, m, seed, query_base, out.data_ptr(), None, None,
                                            export_samples.data_ptr() if export_samples is not None else None,
                                            self._stream()))
        return out


class QueryShardedKDE:
    """Query-sharded mode: rank r evaluates queries [lo_r, hi_r) of every batch against its full
    replica of the dataset and the slices are all-gathered (padded to equal length)."""

    def __init__(self, engine, comm, rank: int, world: int):
        self.engine = engine
        self.comm = comm
        self.rank = int(rank)
        self.world = int(world)
        self.N = engine.n

    def _slice(self, nq):
        return shard_bounds(nq, self.world, self.rank)

    def _gather(self, part, nq, tail_shape=()):
        """all_gather of the per-rank slices (each padded to ceil(nq / world) rows) -> (nq, ...)."""
        import torch

        width = max(1, -(-nq // self.world))
        pad = part.new_zeros((width,) + tuple(tail_shape))
        pad[: part.shape[0]] = part
        allp = self.comm.all_gather(pad)
        rows = []
        for r in range(self.world):
            a, b = shard_bounds(nq, self.world, r)
            rows.append(allp[r][: b - a])
        return torch.cat(rows)

    def naive_kde(self, Q, kernel):
        Qd = self.engine.queries(Q)
        lo, hi = self._slice(Qd.shape[0])
        return self._gather(self.engine.naive(Qd[lo:hi], kernel), Qd.shape[0])

    def knn(self, Q, k):
        if not 1 <= k <= self.N:
            raise ValueError(f"k={k} out of range [1, {self.N}]")
        Qd = self.engine.queries(Q)
        lo, hi = self._slice(Qd.shape[0])
        idx, d2 = self.engine.knn(Qd[lo:hi], k)
        return self._gather(idx, Qd.shape[0], (k,)), self._gather(d2, Qd.shape[0], (k,))

    def deann(self, Q, kernel, k, m, *, seed: int, query_base: int = 0, export_samples: bool = False):
        """Values (nq,) and, with export_samples, the accepted sample ids (nq, m)."""
        if not 0 <= k <= self.N:
            raise ValueError(f"k={k} out of range [0, {self.N}]")
        if m < 0:
            raise ValueError(f"m={m} must be >= 0")
        if m > 0 and k >= self.N:
            raise ValueError("m > 0 requires k + 1 <= n so the remainder is nonempty")
        Qd = self.engine.queries(Q)
        nq = Qd.shape[0]
        lo, hi = self._slice(nq)
        acc = None
        if export_samples and m > 0:
            import torch

            acc = torch.empty((hi - lo, m), dtype=torch.int64, device=Qd.device)
        vals = self.engine.deann(Qd[lo:hi], kernel, k, m, seed, query_base + lo, export_samples=acc)
        vals = self._gather(vals, nq)
        if acc is None:
            return vals
        return vals, self._gather(acc, nq, (m,))

