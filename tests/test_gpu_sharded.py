"""GPU: the per-shard primitives of dataset-sharded mode (two shards on one GPU).

Multi-GPU runs launch one process per GPU (bench.py --gpus N under torchrun);
with one GPU available here, two GpuShardEngine objects on cuda:0 stand in for
two ranks and their partials are combined locally, which is exactly what the
NCCL all_reduce / all_gather do in ShardedKDE (orchestration covered by
tests/test_sharded.py with gloo).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from oracle.philox import IndexReplay, NeighborReplay  # noqa: E402
from paper_2107_02736_b200.sharded import GpuShardEngine, LocalComm, ShardedKDE, shard_bounds  # noqa: E402


@pytest.fixture(scope="module")
def problem():
    rng = np.random.default_rng(17)
    centers = rng.normal(scale=2.0, size=(8, 12))
    X = (centers[rng.integers(0, 8, 9000)] + rng.normal(size=(9000, 12))).astype(np.float32)
    Q = centers[rng.integers(0, 8, 40)] + rng.normal(size=(40, 12))
    engines = []
    for r in range(2):
        lo, hi = shard_bounds(X.shape[0], 2, r)
        engines.append(GpuShardEngine(X[lo:hi], global_offset=lo, global_n=X.shape[0], device=0))
    return X, Q, engines


def test_shard_partial_sums_compose(problem):
    X, Q, (e0, e1) = problem
    for fam, h in [("gaussian", 1.5), ("exponential", 1.0), ("laplacian", 3.0)]:
        spec = g.KernelSpec(fam, h)
        tot = (e0.kde_sums(e0.queries(Q), spec) + e1.kde_sums(e1.queries(Q), spec)) / X.shape[0]
        ref = O.naive_kde(O.Data(X), fam, h, Q)
        assert float(torch.max(torch.abs(tot.cpu() - torch.as_tensor(ref)) / torch.as_tensor(ref))) < 1e-5


def test_shard_knn_merge_is_global(problem):
    X, Q, (e0, e1) = problem
    Qd = e0.queries(Q)
    i0, d0 = e0.knn(Qd, 30)
    i1, d1 = e1.knn(Qd, 30)
    assert int(i1.min()) >= shard_bounds(X.shape[0], 2, 1)[0]
    idx, d2 = e0.merge_topk(torch.stack([i0, i1]), torch.stack([d0, d1]), 30)
    od = O.Data(X)
    for j, q in enumerate(Q):
        ri, rd = O.brute_force_knn(od, q, 30)
        np.testing.assert_array_equal(idx[j].cpu().numpy(), ri)
        np.testing.assert_allclose(d2[j].cpu().numpy(), rd, rtol=1e-6)


@pytest.mark.parametrize("family,h", [("gaussian", 1.5), ("laplacian", 3.0)])
def test_shard_deann_composes_to_single_gpu_and_oracle(problem, family, h):
    X, Q, (e0, e1) = problem
    spec = g.KernelSpec(family, h)
    N, k, m, seed = X.shape[0], 25, 300, 4242
    Qd = e0.queries(Q)
    i0, d0 = e0.knn(Qd, k)
    i1, d1 = e1.knn(Qd, k)
    idx, d2 = e0.merge_topk(torch.stack([i0, i1]), torch.stack([d0, d1]), k)
    z2s = e0.sample_sums(Qd, spec, m, seed, 0, idx) + e1.sample_sums(Qd, spec, m, seed, 0, idx)
    z1s = (e0.row_sums(Qd, spec, idx) + e1.row_sums(Qd, spec, idx)) if family == "laplacian" else None
    val = e0.combine(spec, k, m, d2, z1s, z2s).cpu().numpy()
    single, _, _ = g.deann_arrays(g.Dataset.from_array(X), spec, Q, k, m, seed=seed)
    np.testing.assert_allclose(val, single, rtol=1e-12)
    od = O.Data(X)
    for j, q in enumerate(Q[:10]):
        ri, rd = O.brute_force_knn(od, q, k)
        ref = O.deann(od, family, h, NeighborReplay(ri, rd), q, k, m, rng=IndexReplay(seed, j, N))[0]
        assert val[j] == pytest.approx(ref, rel=1e-12)


def test_sharded_kde_object_single_rank(problem):
    X, Q, _ = problem
    eng = GpuShardEngine(X, global_offset=0, global_n=X.shape[0], device=0)
    sk = ShardedKDE(eng, LocalComm())
    spec = g.KernelSpec("gaussian", 1.5)
    ref = O.naive_kde(O.Data(X), "gaussian", 1.5, Q)
    got = sk.naive_kde(Q, spec).cpu().numpy()
    assert np.max(np.abs(got - ref) / ref) < 1e-5
    v = sk.deann(Q, spec, 10, 100, seed=5).cpu().numpy()
    single, _, _ = g.deann_arrays(g.Dataset.from_array(X), spec, Q, 10, 100, seed=5)
    np.testing.assert_allclose(v, single, rtol=1e-12)


def test_query_sharded_equals_dataset_sharded_gpu(problem):
    """Query-sharded (2 replicas, each a slice of the batch at its global query positions) and
    dataset-sharded (2 row shards, merged k-NN, global Philox stream) give identical k-NN sets,
    identical accepted sample ids and values equal to fp64 summation order."""
    from paper_2107_02736_b200.sharded import GpuReplicaEngine

    X, Q, (e0, e1) = problem
    spec = g.KernelSpec("gaussian", 1.5)
    k, m, seed, base = 20, 200, 31, 5
    Qd = e0.queries(Q)
    nq = Q.shape[0]
    # dataset-sharded
    i0, d0 = e0.knn(Qd, k)
    i1, d1 = e1.knn(Qd, k)
    idx, d2 = e0.merge_topk(torch.stack([i0, i1]), torch.stack([d0, d1]), k)
    acc_ds = torch.empty((nq, m), dtype=torch.int64, device="cuda")
    acc_ds1 = torch.empty((nq, m), dtype=torch.int64, device="cuda")
    z2s = e0.sample_sums(Qd, spec, m, seed, base, idx, export=acc_ds) + \
        e1.sample_sums(Qd, spec, m, seed, base, idx, export=acc_ds1)
    val_ds = e0.combine(spec, k, m, d2, None, z2s)
    assert torch.equal(acc_ds, acc_ds1)  # every rank walks the same global stream
    # query-sharded: two replicas, each its slice
    rep = GpuReplicaEngine(X, device=0)
    vals, accs, idxs = [], [], []
    for r in range(2):
        lo, hi = shard_bounds(nq, 2, r)
        a = torch.empty((hi - lo, m), dtype=torch.int64, device="cuda")
        vals.append(rep.deann(Qd[lo:hi], spec, k, m, seed, base + lo, export_samples=a))
        accs.append(a)
        idxs.append(rep.knn(Qd[lo:hi], k)[0])
    np.testing.assert_array_equal(torch.cat(idxs).cpu().numpy(), idx.cpu().numpy())
    np.testing.assert_array_equal(torch.cat(accs).cpu().numpy(), acc_ds.cpu().numpy())
    np.testing.assert_allclose(torch.cat(vals).cpu().numpy(), val_ds.cpu().numpy(), rtol=1e-12)
