"""Small inputs through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize.py [--pair]

Covers the fused tile sweep in every mode (exact-integer and split3 gaussian, exponential,
TILEMIN / FILTER, the pruned FILTER in tile-major order on >= 512 tiles, the 2-CTA pair
variant with --pair; the norm-column epilogue in the K padding and in the 16-column tail; the
two-precision KDE's fp16 and split3 passes, hot lists, combine and fallback), the L1 kernel, the k-NN selection / fallback / big-k paths, the Philox
sampler, explicit-row evaluation, the permuted sampler, the IVF build and query, and the
shard merge.  Each check also compares against a NumPy reference, so a run that the
sanitizer lets through is still a correct one.
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--pair", action="store_true", help="2-CTA (cta_group::2) tile sweeps (DK_PAIR=1)")
args = ap.parse_args()
if args.pair:
    os.environ["DK_PAIR"] = "1"

import torch  # noqa: E402

import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


rng = np.random.default_rng(0)
# exact-integer tiles (gaussian), split3 (gaussian / exponential), L1
Xi = rng.integers(0, 30, size=(3000, 40)).astype(np.float32)
Qi = rng.integers(0, 30, size=(300, 40)).astype(np.float64)
ds = g.Dataset.from_array(Xi)
check("naive exact-int", np.allclose(g.naive_kde(ds, g.KernelSpec("gaussian", 20.0), Qi).values,
                                      O.naive_kde(O.Data(Xi), "gaussian", 20.0, Qi), rtol=1e-5))
Xf = rng.normal(size=(3000, 24)).astype(np.float32)
Qf = rng.normal(size=(300, 24))
dsf = g.Dataset.from_array(Xf)
odf = O.Data(Xf)
for fam, h in (("gaussian", 2.0), ("exponential", 1.5), ("laplacian", 4.0)):
    check(f"naive {fam}", np.allclose(g.naive_kde(dsf, g.KernelSpec(fam, h), Qf).values,
                                      O.naive_kde(odf, fam, h, Qf), rtol=1e-5))
# k-NN: small (every row a candidate), segmented TILEMIN + FILTER, big k, DEANN / RS / rows
idx, _ = g.knn_batch(dsf, Qf[:50], 20)
check("knn small", all(np.array_equal(idx[j], O.brute_force_knn(odf, Qf[j], 20)[0]) for j in range(50)))
Xm = (rng.normal(scale=4.0, size=(40, 16))[rng.integers(0, 40, 20_000)] + rng.normal(size=(20_000, 16))).astype(
    np.float32)
dsm, odm = g.Dataset.from_array(Xm), O.Data(Xm)
Qm = Xm[rng.integers(0, 20_000, 200)].astype(np.float64) + 0.1
idx, _ = g.knn_batch(dsm, Qm, 30)
check("knn segmented", all(np.array_equal(idx[j], O.brute_force_knn(odm, Qm[j], 30)[0]) for j in range(0, 200, 7)))
idx, _ = g.knn_batch(dsm, Qm[:2], 4500)  # k > 4096: exact fp64 + radix sort path
check("knn big-k", np.array_equal(idx[0], O.brute_force_knn(odm, Qm[0], 4500)[0]))
vals, nbr, smp = g.deann_arrays(dsm, g.KernelSpec("gaussian", 2.0), Qm[:64], 10, 100, seed=3, export_neighbors=True,
                                export_samples=True)
check("deann / sampler", np.all(np.isfinite(vals)) and not np.isin(smp[0], nbr[0]).any())
check("rs", np.isfinite(g.rs_kde(dsm, g.KernelSpec("exponential", 2.0), Qm[0], 50, 7).value))
check("kernel values", np.allclose(g.kernel_from_distance(g.KernelSpec("gaussian", 2.0), np.arange(5.0)),
                                   np.exp(-np.arange(5.0) / 8.0)))
# pruned FILTER (>= 512 tiles): tile-major sweep, device-side ball sort and unit plans
Xp = (rng.normal(scale=5.0, size=(200, 8))[rng.integers(0, 200, 140_000)] + rng.normal(size=(140_000, 8))).astype(
    np.float32)
dsp, odp = g.Dataset.from_array(Xp), O.Data(Xp)
Qp = Xp[rng.integers(0, 140_000, 256)].astype(np.float64) + 0.05
idx, _ = g.knn_batch(dsp, Qp, 16)
check("knn pruned", all(np.array_equal(idx[j], O.brute_force_knn(odp, Qp[j], 16)[0]) for j in range(0, 256, 17)))
# permuted sampler
st = g.RspState.from_dataset(dsm, 5)
check("rsp", np.isfinite(g.rsp_kde(st, g.KernelSpec("gaussian", 2.0), Qm[0], 100).value))
est = g.deann_batch(dsm, g.KernelSpec("gaussian", 2.0), g.BruteForceIndex(dsm), Qm[:16], 8, 64, rsp_state=st)
check("deannp", all(np.isfinite(e.value) for e in est))
# IVF
ivf = g.IvfAnnIndex.build(dsm, 32, 1, 4)
nl = ivf.query(Qm[0], 10)
check("ivf query", len(nl.indices) == 10)
est = g.deann_batch(dsm, g.KernelSpec("gaussian", 2.0), ivf, Qm[:32], 10, 100, rng=g.PhiloxSampler(1))
check("deann ivf", all(np.isfinite(e.value) for e in est))
# shard merge
from paper_2107_02736_b200.sharded import GpuShardEngine  # noqa: E402

e0 = GpuShardEngine(Xm[:9000], global_offset=0, global_n=20_000)
e1 = GpuShardEngine(Xm[9000:], global_offset=9000, global_n=20_000)
Qd = e0.queries(Qm[:32])
a, b = e0.knn(Qd, 12), e1.knn(Qd, 12)
mi, _ = e0.merge_topk(torch.stack([a[0], b[0]]), torch.stack([a[1], b[1]]), 12)
check("merge topk", np.array_equal(mi.cpu().numpy()[0], O.brute_force_knn(odm, Qm[0], 12)[0]))
# norm columns in the 16-column tail (d = 128 integer rows) and in the K padding (d = 100)
for dd in (128, 100):
    Xi = rng.integers(0, 64, size=(3000, dd)).astype(np.float32)
    Qi = rng.integers(0, 64, size=(40, dd)).astype(np.float64)
    got = g.naive_kde(g.Dataset.from_array(Xi), g.KernelSpec("gaussian", 60.0), Qi).values
    check(f"norm columns d={dd}", np.max(np.abs(got - O.naive_kde(O.Data(Xi), "gaussian", 60.0, Qi)) /
                                        O.naive_kde(O.Data(Xi), "gaussian", 60.0, Qi)) < 2e-6)
# two-precision exact KDE (>= 512 tiles, >= 2,048 queries), with forced fallbacks for a few queries
import workloads  # noqa: E402

Xh = workloads._c3_rows(3, 140_000)
Qh = workloads._c3_rows(4, 2048).astype(np.float64)
Qh[:3] = rng.standard_normal((3, Xh.shape[1]))  # unit directions far from every cluster: the fp16
Qh[:3] /= np.linalg.norm(Qh[:3], axis=1, keepdims=True)  # bound fails -> split3 fallback
dsh = g.Dataset.from_array(Xh)
vh = g.naive_kde(dsh, g.KernelSpec("gaussian", 0.2239), Qh).values
refh = O.naive_kde(O.Data(Xh), "gaussian", 0.2239, Qh[:8])
check("two-precision KDE", float(np.max(np.abs(vh[:8] - refh) / refh)) < 1e-5)
torch.cuda.synchronize()
print("sanitize workload done", flush=True)
