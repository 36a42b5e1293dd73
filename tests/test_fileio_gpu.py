"""GPU side of the format layer: the device CRC-32, the codes writer for CUDA
codes, and the streaming fvecs/bvecs -> PQCD encoder, against files written by
the reference's own writers (tests/golden/io_golden.npz) and its reader errors."""

import zlib

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

IO = golden("io_golden.npz")


@pytest.fixture(scope="module")
def P():
    import paper_2605_25521_b200 as P
    return P


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1023, 1024, 1025, 262143, 262144, 262145, 3 * 262144 + 11,
                               5_000_003])
@pytest.mark.parametrize("crc_in", [0, 0xDEADBEEF])
def test_crc32_device_matches_zlib(P, n, crc_in):
    import torch
    rng = np.random.default_rng(n + 1)
    data = rng.integers(0, 256, n, dtype=np.uint8)
    got = P.crc32_device(torch.from_numpy(data).cuda(), crc_in)
    assert got == zlib.crc32(data.tobytes(), crc_in)


def test_crc32_device_unaligned_view(P):
    import torch
    data = np.random.default_rng(9).integers(0, 256, 100_003, dtype=np.uint8)
    t = torch.from_numpy(data).cuda()
    assert P.crc32_device(t[3:]) == zlib.crc32(data[3:].tobytes())


@pytest.mark.parametrize("key,k", [("pqcd8", 200), ("pqcd16", 1000)])
def test_write_codes_from_device(P, tmp_path, key, k):
    import torch
    codes = IO[f"{key}/codes"]
    p = tmp_path / "c.pqcd"
    P.write_codes(p, torch.from_numpy(codes).cuda(), k=k)
    assert p.read_bytes() == IO[f"{key}/bytes"].tobytes()


def _codebooks(P, rm):
    return [P.Codebook.from_rowmajor(j, rm[j]) for j in range(rm.shape[0])]


@pytest.mark.parametrize("name,ext", [("file_f32", "fvecs"), ("file_u8", "bvecs")])
@pytest.mark.parametrize("mode", ["auto", "exact", "guarded"])
@pytest.mark.parametrize("batch_rows,streams", [(None, 3), (333, 1), (333, 3), (4096, 2)])
def test_encode_file_matches_reference_bytes(P, tmp_path, name, ext, mode, batch_rows, streams):
    src = tmp_path / f"in.{ext}"
    src.write_bytes(IO[f"{name}/vecs_bytes"].tobytes())
    out = tmp_path / "out.pqcd"
    plan = P.ExecutionPlan(mode=mode, batch_rows=batch_rows, streams=streams)
    info = P.encode_file(src, _codebooks(P, IO[f"{name}/rowmajor"]), out, plan)
    assert info["n"] == IO[f"{name}/X"].shape[0]
    assert out.read_bytes() == IO[f"{name}/pqcd_bytes"].tobytes()


def test_encode_file_equals_in_memory_path(P, tmp_path, oracle):
    """A larger fvecs file: the file encoder's codes = encode_dataset's = the oracle's."""
    rng = np.random.default_rng(4)
    X = rng.standard_normal((50_000, 128)).astype(np.float32)
    rm = (rng.standard_normal((16, 256, 8)) * 0.8).astype(np.float32)
    cbs = _codebooks(P, rm)
    src, out = tmp_path / "big.fvecs", tmp_path / "big.pqcd"
    P.write_fvecs(src, X)
    P.encode_file(src, cbs, out, P.ExecutionPlan(batch_rows=7000))
    got = P.read_codes(out)
    cs = P.CodebookSet.from_codebooks(cbs)
    want = oracle.encode(X, cs.rowmajor, cs.biases, oracle.VARIANT_REFORM)
    assert got.codes.tobytes() == want.tobytes()
    assert got.codes.tobytes() == P.encode_dataset(X, cbs).codes.tobytes()


def test_encode_file_errors_match_reference_reader(P, tmp_path):
    rm = (np.random.default_rng(1).standard_normal((1, 256, 2))).astype(np.float32)
    cbs = _codebooks(P, rm)
    for key, msg, off in zip(IO["err/keys"], IO["err/messages"], IO["err/offsets"]):
        src = tmp_path / f"{key}.fvecs"
        src.write_bytes(IO[f"err/{key}/bytes"].tobytes())
        out = tmp_path / f"{key}.pqcd"
        with pytest.raises(P.FormatError) as ei:
            P.encode_file(src, cbs, out)
        assert str(ei.value).replace(str(src), "<path>") == str(msg), key
        assert ei.value.offset == int(off), key
        assert not out.exists(), key


def test_encode_file_error_precedence(P, tmp_path):
    """A bad header after a non-finite value wins (the reference walks every
    record before checking values), however the batches fall."""
    import struct
    cbs = _codebooks(P, np.random.default_rng(2).standard_normal((1, 256, 2)).astype(np.float32))
    recs = [struct.pack("<i2f", 2, 1.0, 2.0)] * 50
    recs[3] = struct.pack("<i2f", 2, float("nan"), 2.0)
    recs[40] = struct.pack("<i2f", 5, 1.0, 2.0)
    src = tmp_path / "x.fvecs"
    src.write_bytes(b"".join(recs))
    with pytest.raises(P.FormatError, match="inconsistent fvecs record length 5") as ei:
        P.encode_file(src, cbs, tmp_path / "o.pqcd", P.ExecutionPlan(batch_rows=8))
    assert ei.value.offset == 40 * 12
    recs[40] = struct.pack("<i2f", 2, 1.0, 2.0)
    src.write_bytes(b"".join(recs))
    with pytest.raises(P.FormatError, match="non-finite") as ei:
        P.encode_file(src, cbs, tmp_path / "o.pqcd", P.ExecutionPlan(batch_rows=8))
    assert ei.value.offset == 3 * 12 + 4


def test_encode_file_dimension_mismatch(P, tmp_path):
    src = tmp_path / "x.fvecs"
    P.write_fvecs(src, np.ones((4, 6), np.float32))
    cbs = _codebooks(P, np.random.default_rng(3).standard_normal((2, 256, 2)).astype(np.float32))
    with pytest.raises(P.ConfigError, match="dimensionality 6"):
        P.encode_file(src, cbs, tmp_path / "o.pqcd")


def test_encode_file_wide_codes_generic_shape(P, tmp_path):
    """k = 1000 (uint16 codes, generic kernel) on d_sub = 3 rows: the streamed file equals
    write_codes(encode_dataset(...)) byte for byte."""
    rng = np.random.default_rng(21)
    X = rng.standard_normal((5003, 12)).astype(np.float32)
    rm = rng.standard_normal((4, 1000, 3)).astype(np.float32)
    cbs = _codebooks(P, rm)
    src, out, ref = tmp_path / "w.fvecs", tmp_path / "w.pqcd", tmp_path / "ref.pqcd"
    P.write_fvecs(src, X)
    P.encode_file(src, cbs, out, P.ExecutionPlan(batch_rows=1500))
    P.write_codes(ref, P.encode_dataset(X, cbs))
    assert out.read_bytes() == ref.read_bytes()
    assert P.read_codes(out).codes.dtype == np.uint16
