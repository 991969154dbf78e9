"""DEANN1 dataset files against the reference's own save/load.

Goldens (tests/golden/make_golden.py) hold the bytes the reference's ``save``
writes, the norms its ``load`` computes and the DatasetFormatError messages it
raises for malformed files.  Header validation runs in the C-ABI without a
GPU; the device upload (dk_fit_file) is covered by the ``gpu`` tests.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2107_02736_b200 as g
from dk_testutil import malformed_files


def _golden_rows(golden):
    raw = golden["file_bytes"].tobytes()
    n, d = np.frombuffer(raw[8:16], "<u4")
    return raw, np.frombuffer(raw[16:], "<f4").reshape(int(n), int(d))


def test_save_is_bit_identical_to_reference(golden, tmp_path):
    raw, X = _golden_rows(golden)
    p = tmp_path / "ours.bin"
    g.save(X, p)
    assert p.read_bytes() == raw


def test_file_info_reads_the_reference_header(golden, tmp_path):
    raw, X = _golden_rows(golden)
    p = tmp_path / "ref.bin"
    p.write_bytes(raw)
    assert g.file_info(p) == X.shape


@pytest.mark.parametrize("i", range(9))
def test_malformed_files_raise_the_reference_messages(golden, tmp_path, i):
    raw, _ = _golden_rows(golden)
    name, data = malformed_files(raw)[i]
    assert str(golden["file_bad_names"][i]) == name
    p = tmp_path / name
    p.write_bytes(data)
    with pytest.raises(g.DatasetFormatError) as exc:
        g.file_info(p)
    assert str(exc.value).replace(str(p), "<P>") == str(golden["file_bad_msgs"][i])
    assert isinstance(exc.value, ValueError)


def test_missing_file_is_file_not_found(tmp_path):
    with pytest.raises(FileNotFoundError):
        g.file_info(tmp_path / "nope.bin")
    with pytest.raises(FileNotFoundError):
        g.load(tmp_path / "nope.bin")


def test_unknown_format(tmp_path):
    with pytest.raises(ValueError):
        g.load(tmp_path / "x", fmt="parquet")
    with pytest.raises(ValueError):
        g.save(np.zeros((2, 2), np.float32), tmp_path / "x", fmt="parquet")


def test_csv_parse_errors_match_reference_format(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("1,2,3\n4,5\n")
    with pytest.raises(g.DatasetFormatError, match=r"line 2 has 2 fields, expected 3"):
        g.load(p, fmt="csv")
    p.write_text("\n\n")
    with pytest.raises(g.DatasetFormatError, match="no data rows"):
        g.load(p, fmt="csv")
    p.write_text("1,abc\n")
    with pytest.raises(g.DatasetFormatError, match="line 1"):
        g.load(p, fmt="csv")


# ------------------------------------------------------------------ GPU upload


@pytest.mark.gpu
def test_load_binary_matches_reference_norms_and_rows(golden, tmp_path):
    raw, X = _golden_rows(golden)
    p = tmp_path / "ref.bin"
    p.write_bytes(raw)
    ds = g.load(p)
    assert ds.n == X.shape[0] and ds.d == X.shape[1]
    assert ds.data.tobytes() == X.tobytes()
    np.testing.assert_allclose(ds.sq_norms, golden["file_sq_norms"], rtol=1e-15, atol=0)
    ref = g.Dataset.from_array(X)
    Q = np.random.default_rng(3).normal(size=(9, X.shape[1]))
    for fam in ("gaussian", "exponential", "laplacian"):
        a = g.naive_kde(ds, g.KernelSpec(fam, 2.0), Q).values
        b = g.naive_kde(ref, g.KernelSpec(fam, 2.0), Q).values
        np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_load_csv_roundtrip(tmp_path):
    X = np.random.default_rng(4).normal(size=(11, 4)).astype(np.float32)
    p = tmp_path / "x.csv"
    g.save(X, p, fmt="csv")
    ds = g.load(p, fmt="csv")
    np.testing.assert_array_equal(ds.data, X)  # %.9g round-trips float32


@pytest.mark.gpu
def test_streamed_upload_of_a_multi_chunk_file(tmp_path):
    # 150 MB: several 16 MB pinned chunks per reader group, a ragged last chunk
    rng = np.random.default_rng(5)
    X = rng.normal(size=(384_001, 100)).astype(np.float32)
    p = tmp_path / "big.bin"
    g.save(X, p)
    ds = g.load(p)
    ref = np.einsum("ij,ij->i", X.astype(np.float64), X.astype(np.float64))
    np.testing.assert_allclose(ds.sq_norms, ref, rtol=1e-13)
    idx, d2 = g.knn_batch(ds, X[[0, 191_000, 384_000]].astype(np.float64), 1)
    assert idx[:, 0].tolist() == [0, 191_000, 384_000]


@pytest.mark.gpu
def test_row_range_shards_reassemble_the_file(tmp_path):
    from paper_2107_02736_b200.sharded import GpuShardEngine, shard_bounds

    X = np.random.default_rng(6).normal(size=(5003, 12)).astype(np.float32)
    p = tmp_path / "s.bin"
    g.save(X, p)
    Q = np.random.default_rng(7).normal(size=(6, 12))
    full = g.naive_kde(g.Dataset.from_array(X), g.KernelSpec("gaussian", 1.5), Q).values * X.shape[0]
    total = np.zeros(len(Q))
    for r in range(3):
        eng = GpuShardEngine.from_file(p, 3, r)
        lo, hi = shard_bounds(X.shape[0], 3, r)
        assert (eng.global_offset, eng.n_local, eng.global_n) == (lo, hi - lo, X.shape[0])
        assert eng.ds.data.tobytes() == X[lo:hi].tobytes()
        total += eng.kde_sums(eng.queries(Q), g.KernelSpec("gaussian", 1.5)).cpu().numpy()
    np.testing.assert_allclose(total, full, rtol=1e-5)  # per-shard encodings round differently (KDE_RTOL)
    with pytest.raises(ValueError):
        g.load(p, rows=(5000, 10))
