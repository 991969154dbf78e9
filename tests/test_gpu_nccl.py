"""GPU, >= 2 devices: dataset-sharded and query-sharded modes end to end over NCCL.

One process per GPU (torch.multiprocessing, backend "nccl"): GpuShardEngine shards
+ TorchComm for dataset-sharded mode, GpuReplicaEngine replicas for query-sharded
mode, both against the single-GPU fused path on rank 0.  Skipped when fewer than
two GPUs are visible (the orchestration itself is covered with gloo on CPU in
tests/test_sharded.py, the per-shard kernels on one GPU in tests/test_gpu_sharded.py).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _problem():
    rng = np.random.default_rng(23)
    centers = rng.normal(scale=3.0, size=(16, 24))
    X = (centers[rng.integers(0, 16, 20_000)] + rng.normal(size=(20_000, 24))).astype(np.float32)
    Q = centers[rng.integers(0, 16, 300)] + rng.normal(size=(300, 24))
    return X, Q


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_2107_02736_b200 as g
        from paper_2107_02736_b200.sharded import (GpuReplicaEngine, GpuShardEngine, QueryShardedKDE, ShardedKDE,
                                                   TorchComm, shard_bounds)

        X, Q = _problem()
        spec = g.KernelSpec("gaussian", 2.5)
        lo, hi = shard_bounds(X.shape[0], world, rank)
        sk = ShardedKDE(GpuShardEngine(X[lo:hi], global_offset=lo, global_n=X.shape[0], device=rank), TorchComm())
        qs = QueryShardedKDE(GpuReplicaEngine(X, device=rank), TorchComm(), rank, world)
        out = {"ds_naive": sk.naive_kde(Q, spec).cpu().numpy()}
        i, d = sk.knn(Q, 30)
        out["ds_idx"], out["ds_d2"] = i.cpu().numpy(), d.cpu().numpy()
        acc = torch.empty((Q.shape[0], 400), dtype=torch.int64, device=f"cuda:{rank}")
        out["ds_deann"] = sk.deann(Q, spec, 30, 400, seed=9, query_base=2, export_samples=acc).cpu().numpy()
        out["ds_acc"] = acc.cpu().numpy()
        out["qs_naive"] = qs.naive_kde(Q, spec).cpu().numpy()
        i, d = qs.knn(Q, 30)
        out["qs_idx"], out["qs_d2"] = i.cpu().numpy(), d.cpu().numpy()
        v, a = qs.deann(Q, spec, 30, 400, seed=9, query_base=2, export_samples=True)
        out["qs_deann"], out["qs_acc"] = v.cpu().numpy(), a.cpu().numpy()
        if rank == 0:
            ds = g.Dataset.from_array(X, device=0)
            out["one_naive"] = g.naive_kde(ds, spec, Q).values
            out["one_idx"], out["one_d2"] = g.knn_batch(ds, Q, 30)
            out["one_deann"], _, out["one_acc"] = g.deann_arrays(ds, spec, Q, 30, 400, seed=9, query_base=2,
                                                                 export_samples=True)
            results.update(out)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_results():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    return dict(results)


def test_dataset_sharded_equals_single_gpu(nccl_results):
    r = nccl_results
    np.testing.assert_allclose(r["ds_naive"], r["one_naive"], rtol=1e-6)
    np.testing.assert_array_equal(r["ds_idx"], r["one_idx"])
    np.testing.assert_array_equal(r["ds_acc"], r["one_acc"])
    np.testing.assert_allclose(r["ds_deann"], r["one_deann"], rtol=1e-12)


def test_query_sharded_equals_single_gpu(nccl_results):
    r = nccl_results
    np.testing.assert_allclose(r["qs_naive"], r["one_naive"], rtol=1e-12)  # column chunking follows the batch size
    np.testing.assert_array_equal(r["qs_idx"], r["one_idx"])
    np.testing.assert_array_equal(r["qs_acc"], r["one_acc"])
    np.testing.assert_array_equal(r["qs_deann"], r["one_deann"])
