"""Generate the golden fixtures by importing the REAL reference package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Runs only in the build container (the reference is not on the GPU box); the
outputs (tests/golden/*.npz) are committed.  Every value below is produced by
the reference's own functions (deann.naive_kde, deann.brute_force_knn,
deann.rs_kde, deann.deann, deann.kernel_from_distance) — the oracle restatement
(oracle/deann_oracle.py) and the GPU path are both checked against them.
Sampling goldens feed the reference a replay of the GPU's Philox stream
(oracle.philox.IndexReplay) through its public `rng=` argument, so they pin the
"first m accepted draws" semantics of _rs_excluding (estimators.py:203-233).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "tests"))

import deann  # noqa: E402  (the reference)

from oracle.philox import IndexReplay  # noqa: E402
from dk_testutil import malformed_files  # noqa: E402


class _Fixed:
    def __init__(self, nl):
        self.nl = nl

    def query(self, y, k):
        return self.nl


def _random_dataset(n, d, seed):
    return np.random.default_rng(seed).normal(size=(n, d)).astype(np.float32)


def main():
    out = {}
    # --- kernels.py known answers (test_kernels.py:15-50)
    ks = deann.KernelSpec
    out["kat_values"] = np.array([
        deann.kernel_from_distance(ks("gaussian", 1.0), 0.0),
        deann.kernel_from_distance(ks("exponential", 2.0), 2.0),
        deann.kernel_from_distance(ks("gaussian", 0.5), 3.0),
        deann.kernel_pair(ks("exponential", 1.0), [0.0, 0.0], [3.0, 4.0]),
        deann.kernel_pair(ks("laplacian", 2.0), [1.0, 1.0], [2.0, 3.0]),
    ])

    # --- naive_kde on random datasets, all families (test_estimators.py:55-63 pattern)
    cases = []
    for i, (n, d, fam, h) in enumerate([(500, 10, "gaussian", 1.0), (500, 10, "exponential", 1.7),
                                        (500, 10, "laplacian", 2.2), (2000, 37, "gaussian", 3.0),
                                        (1500, 3, "exponential", 0.4), (300, 130, "laplacian", 40.0)]):
        X = _random_dataset(n, d, 100 + i)
        Q = np.random.default_rng(200 + i).normal(size=(16, d))
        ds = deann.Dataset.from_array(X)
        v = deann.naive_kde(ds, ks(fam, h), Q).values
        out[f"naive_{i}_X"], out[f"naive_{i}_Q"], out[f"naive_{i}_v"] = X, Q, v
        out[f"naive_{i}_meta"] = np.array([h, ["gaussian", "exponential", "laplacian"].index(fam)])
        cases.append(i)
    out["naive_cases"] = np.array(cases)

    # --- acceptance 1 instances (test_acceptance.py:48-86)
    rng = np.random.default_rng(11)
    fams = ("gaussian", "exponential", "laplacian")
    for i in range(20):
        n = int(rng.integers(50, 1001))
        d = int(rng.integers(2, 33))
        X = rng.normal(size=(n, d)).astype(np.float32)
        q = rng.normal(size=d)
        h = 0.5 + (i % 5) * 0.6
        fam = fams[i % 3]
        v = deann.naive_kde(deann.Dataset.from_array(X), ks(fam, h), q.reshape(1, -1)).values[0]
        out[f"acc1_{i}_X"], out[f"acc1_{i}_q"], out[f"acc1_{i}_v"] = X, q, np.array([v, h, i % 3])

    # --- brute-force k-NN incl. ties (test_ann.py:42-64)
    X = _random_dataset(300, 8, 1)
    X[50:60] = X[40]          # duplicate rows -> exact ties resolved by lower index
    Q = np.random.default_rng(2).normal(size=(12, 8))
    Q[0] = X[40]
    ds = deann.Dataset.from_array(X)
    idx, d2 = [], []
    for q in Q:
        nl = deann.brute_force_knn(ds, q, 25)
        idx.append(nl.indices)
        d2.append(nl.sq_distances)
    out["knn_X"], out["knn_Q"], out["knn_idx"], out["knn_d2"] = X, Q, np.array(idx), np.array(d2)

    # --- rs_kde / deann under a replayed Philox stream (reference consumes rng.integers)
    X = _random_dataset(400, 6, 3)
    Q = np.random.default_rng(4).normal(size=(6, 6))
    ds = deann.Dataset.from_array(X)
    bf = deann.BruteForceIndex(ds)
    rs_vals, de_vals, de_nbr = [], [], []
    seed = 0x1234_5678_9ABC
    for j, q in enumerate(Q):
        for fi, (fam, h) in enumerate([("gaussian", 1.3), ("exponential", 1.1), ("laplacian", 2.5)]):
            rs_vals.append(deann.rs_kde(ds, ks(fam, h), q, 37, IndexReplay(seed, j, 400)).value)
            est = deann.deann(ds, ks(fam, h), bf, q, 15, 50, rng=IndexReplay(seed + 1, j, 400))
            de_vals.append(est.value)
        de_nbr.append(bf.query(q, 15).indices)
    out["samp_X"], out["samp_Q"] = X, Q
    out["samp_rs"], out["samp_deann"], out["samp_nbr"] = np.array(rs_vals), np.array(de_vals), np.array(de_nbr)
    out["samp_seed"] = np.array([seed], dtype=np.uint64)
    # the Philox stream itself (first 64 draws of query 0 / 5 over n=400 and n=1.2M)
    out["philox_q0"] = IndexReplay(seed, 0, 400).integers(0, 400, 64)
    out["philox_q5_big"] = IndexReplay(seed, 5, 1_200_000).integers(0, 1_200_000, 64)

    # --- deann limits (test_estimators.py:176-201, acceptance 2)
    X = _random_dataset(80, 6, 17)
    q = np.random.default_rng(18).normal(size=6)
    ds = deann.Dataset.from_array(X)
    out["lim_X"], out["lim_q"] = X, q
    out["lim_naive"] = np.array([deann.naive_kde(ds, ks("gaussian", 1.4), q.reshape(1, -1)).values[0]])
    out["lim_kn"] = np.array([deann.deann(ds, ks("gaussian", 1.4), deann.BruteForceIndex(ds), q, 80, 0).value])

    # --- permuted sampler: rsp_kde sequences, DEANNP with brute force, deann_batch cursors
    X = _random_dataset(300, 5, 50)
    Q = np.random.default_rng(51).normal(size=(5, 5))
    ds = deann.Dataset.from_array(X)
    bf = deann.BruteForceIndex(ds)
    rsp_vals, rsp_cur, dp_vals, dp_cur, dp_used = [], [], [], [], []
    for fi, (fam, h) in enumerate([("gaussian", 1.1), ("exponential", 0.8), ("laplacian", 2.3)]):
        st = deann.RspState.from_dataset(ds, 60 + fi, cursor=37 * fi)
        for j, q in enumerate(Q):
            rsp_vals.append(deann.rsp_kde(st, ks(fam, h), q, [17, 100, 299, 1, 64][j]).value)
            rsp_cur.append(st.cursor)
        st = deann.RspState.from_dataset(ds, 70 + fi, cursor=290)
        for j, q in enumerate(Q):
            e = deann.deann(ds, ks(fam, h), bf, q, [10, 0, 25, 299, 5][j], [40, 30, 280, 1, 0][j], rsp_state=st)
            dp_vals.append(e.value)
            dp_used.append([e.samples_used, int(e.clamped), int(e.truncated)])
            dp_cur.append(st.cursor)
    shared = deann.RspState.from_dataset(ds, 80, cursor=123)
    batch = deann.deann_batch(ds, ks("gaussian", 1.1), bf, Q, 12, 50, rsp_state=shared)
    indep = deann.deann_batch(ds, ks("gaussian", 1.1), bf, Q, 12, 50, rsp_state=shared, independent_cursors=True)
    out["rsp_X"], out["rsp_Q"] = X, Q
    out["rsp_vals"], out["rsp_cursor"] = np.array(rsp_vals), np.array(rsp_cur)
    out["dp_vals"], out["dp_cursor"], out["dp_used"] = np.array(dp_vals), np.array(dp_cur), np.array(dp_used)
    out["dp_batch"] = np.array([e.value for e in batch])
    out["dp_batch_cursor"] = np.array([shared.cursor])
    out["dp_indep"] = np.array([e.value for e in indep])
    out["rsp_perm80"] = deann.RspState.from_dataset(ds, 80).permuted.permutation.copy()

    # --- DEANN1 files (row f4): reference save bytes, load norms, and its error messages
    import tempfile

    X = _random_dataset(37, 7, 90)
    X[0, :3] = [-0.0, 1e-40, 3.0e38]  # signed zero, a denormal, a large finite value
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "ds.bin")
        deann.save(deann.Dataset.from_array(X), p)
        raw = open(p, "rb").read()
        out["file_bytes"] = np.frombuffer(raw, np.uint8).copy()
        out["file_sq_norms"] = deann.load(p).sq_norms.copy()
        cases = malformed_files(raw)
        msgs = []
        for name, data in cases:
            q = os.path.join(td, name)
            open(q, "wb").write(data)
            try:
                deann.load(q)
                msgs.append("")
            except deann.DatasetFormatError as exc:
                msgs.append(str(exc).replace(q, "<P>"))
        out["file_bad_names"] = np.array([c[0] for c in cases])
        out["file_bad_msgs"] = np.array(msgs)

    # --- inverted file (row f3): ivf_build / ivf_query / IvfAnnIndex / save_ivf_index
    for tag, (n, d, C, seed) in {"ivf_a": (500, 6, 12, 3), "ivf_b": (20_000, 16, 64, 7)}.items():
        X = np.random.default_rng(seed).normal(size=(n, d)).astype(np.float32)
        Q = np.random.default_rng(seed + 1).normal(size=(8, d))
        ds = deann.Dataset.from_array(X)
        index = deann.ivf_build(ds, C, seed=seed)
        out[f"{tag}_cent"] = index.centroids.copy()
        out[f"{tag}_rows"] = np.concatenate(index.assignments).astype(np.int64)
        out[f"{tag}_off"] = np.concatenate([[0], np.cumsum([len(a) for a in index.assignments])]).astype(np.int64)
        probes = [1, 2, 5, C]
        qi, qd, ai, ad = [], [], [], []
        for p_ in probes:
            ann = deann.IvfAnnIndex(ds, index, p_)
            for q in Q:
                nl = deann.ivf_query(index, ds, q, 10, p_)
                qi.append(np.pad(nl.indices, (0, 10 - len(nl)), constant_values=-1))
                qd.append(np.pad(nl.sq_distances, (0, 10 - len(nl)), constant_values=np.inf))
                nl = ann.query(q, 10)
                ai.append(np.pad(nl.indices, (0, 10 - len(nl)), constant_values=-1))
                ad.append(np.pad(nl.sq_distances, (0, 10 - len(nl)), constant_values=np.inf))
        out[f"{tag}_probes"] = np.array(probes)
        out[f"{tag}_q_idx"], out[f"{tag}_q_d2"] = np.array(qi), np.array(qd)
        out[f"{tag}_ann_idx"], out[f"{tag}_ann_d2"] = np.array(ai), np.array(ad)
        if tag == "ivf_a":
            with tempfile.TemporaryDirectory() as td:
                p = os.path.join(td, "ivf.bin")
                deann.save_ivf_index(index, p)
                out["ivf_a_file"] = np.frombuffer(open(p, "rb").read(), np.uint8).copy()

    # --- IvfAnnIndex fp32-ranking semantics (ann.py:276-316) on engineered near-ties: integer rows
    # with |x|^2 > 2^24, so the fp32 keys norms32 - 2 dot collide for rows whose exact (fp64)
    # distances differ by 1 (norms32 rounds to even) while every fp32 / fp64 operation stays exact
    # in any summation order; the reference then selects by list position among equal fp32 keys
    # where exact ranking would select by distance.  Inputs and the reference's answers.
    for tag, (n, d, C, seed) in {"ivf_t1": (600, 4, 8, 11), "ivf_t2": (3000, 6, 24, 12)}.items():
        rng = np.random.default_rng(seed)
        X = rng.integers(0, 6, size=(n, d)).astype(np.float32)
        X[:, 0] = rng.integers(5000, 5040, size=n)
        Q = rng.integers(0, 4, size=(12, d)).astype(np.float64)
        ds = deann.Dataset.from_array(X)
        index = deann.ivf_build(ds, C, seed=seed)
        out[f"{tag}_X"], out[f"{tag}_Q"] = X, Q
        out[f"{tag}_cent"] = index.centroids.copy()
        out[f"{tag}_rows"] = np.concatenate(index.assignments).astype(np.int64)
        out[f"{tag}_off"] = np.concatenate([[0], np.cumsum([len(a) for a in index.assignments])]).astype(np.int64)
        probes = [1, 3, C]
        ai, ad = [], []
        for p_ in probes:
            ann = deann.IvfAnnIndex(ds, index, p_)
            for q in Q:
                nl = ann.query(q, 10)
                ai.append(np.pad(nl.indices, (0, 10 - len(nl)), constant_values=-1))
                ad.append(np.pad(nl.sq_distances, (0, 10 - len(nl)), constant_values=np.inf))
        out[f"{tag}_probes"] = np.array(probes)
        out[f"{tag}_ann_idx"], out[f"{tag}_ann_d2"] = np.array(ai), np.array(ad)

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
