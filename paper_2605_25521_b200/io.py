"""Vector files and the versioned binary containers around the encode path.

Host-side mirror of the reference's formats (/root/reference/pkg/src/cspq/io.py):
same names, same layouts, same FormatError messages and byte offsets.

* fvecs / ivecs / bvecs (io.py:35-121): each record is a little-endian int32
  count d followed by d float32 / int32 / uint8 values; every record must
  share one d.  Readers reject rather than repair.
* PQCB codebooks (io.py:153-210): magic | version u32 | d u32 | m u32 |
  sub_dim u32 | k u32 | m x (k x sub f32 centroids) | m x (k f32 biases) |
  crc32 u32 of everything after the magic.  Stored biases are authoritative.
* PQCD codes (io.py:213-244): magic | version u32 | n u64 | m u32 | k u32 |
  width u32 | n x m codes (u8 when k <= 256 else u16 le) | crc32 u32.

GPU additions (include/cspq_b200.h, csrc/fileio.cu):
* ``encode_file`` streams an fvecs/bvecs file straight into a PQCD file on the
  GPU (read_fvecs + encode_dataset + write_codes without materialising the
  dataset; bvecs rows stay uint8 end to end);
* ``crc32_device`` / ``write_codes`` on CUDA codes checksum the codes where
  they live.
"""

from __future__ import annotations

import ctypes
import os
import struct
import zlib
from pathlib import Path

import numpy as np

from . import _native as N
from .core import Codebook, ConfigError, FormatError, PQCodes, VectorDataset, _readonly

__all__ = [
    "read_fvecs", "write_fvecs", "read_ivecs", "write_ivecs", "read_bvecs", "write_bvecs", "synth_dataset",
    "write_codebooks", "read_codebooks", "write_codes", "read_codes", "encode_file", "crc32_device",
    "CODEBOOK_MAGIC", "CODES_MAGIC", "FORMAT_VERSION",
]

CODEBOOK_MAGIC = b"PQCB"
CODES_MAGIC = b"PQCD"
FORMAT_VERSION = 1
_CODES_HEADER = struct.Struct("<IQIII")   # version, n, m, k, width
_CODEBOOK_HEADER = struct.Struct("<IIIII")  # version, d, m, sub_dim, k


# ---------------------------------------------------------------- texmex records

def _walk_error(raw: np.ndarray, itemsize: int, kind: str) -> FormatError:
    """The first problem a sequential record walk meets (io.py:35-62)."""
    size = raw.shape[0]
    off = 0
    first = None
    while off < size:
        if off + 4 > size:
            return FormatError(f"truncated {kind} record header", offset=off)
        d = int(raw[off:off + 4].view("<i4")[0])
        if d <= 0:
            return FormatError(f"non-positive {kind} record length {d}", offset=off)
        if first is None:
            first = d
        elif d != first:
            return FormatError(f"inconsistent {kind} record length {d} (expected {first})", offset=off)
        if off + 4 + d * itemsize > size:
            return FormatError(f"truncated {kind} record body", offset=off + 4)
        off += 4 + d * itemsize
    raise AssertionError("no record error found")


def _records(path, value_dtype: np.dtype, kind: str) -> np.ndarray:
    """(n, d) values of a record file: one vectorised header check; the exact
    sequential walk only runs to name the first error."""
    raw = np.fromfile(path, dtype=np.uint8)
    if raw.shape[0] == 0:
        raise FormatError(f"empty dataset: {path}", offset=0)
    item = value_dtype.itemsize
    if raw.shape[0] < 4:
        raise _walk_error(raw, item, kind)
    d = int(raw[:4].view("<i4")[0])
    rec = 4 + d * item if d > 0 else 0
    if d <= 0 or raw.shape[0] % rec:
        raise _walk_error(raw, item, kind)
    table = raw.reshape(-1, rec)
    heads = np.ascontiguousarray(table[:, :4]).view("<i4").ravel()
    if not np.all(heads == d):
        raise _walk_error(raw, item, kind)
    return np.ascontiguousarray(table[:, 4:]).view(value_dtype)


def read_fvecs(path) -> VectorDataset:
    """Little-endian float32 vectors; all records share one d; non-finite
    values are rejected with their byte offset (io.py:65-77)."""
    data = _records(path, np.dtype("<f4"), "fvecs")
    bad = ~np.isfinite(data)
    if bad.any():
        row, col = divmod(int(np.flatnonzero(bad.ravel())[0]), data.shape[1])
        raise FormatError("non-finite value in fvecs payload", offset=row * (4 + data.shape[1] * 4) + 4 + col * 4)
    return VectorDataset(data=data.astype(np.float32), source=str(path))


def _write_records(path, mat: np.ndarray, value_dtype: str) -> None:
    n, d = mat.shape
    rec = np.empty(n, dtype=np.dtype([("d", "<i4"), ("v", value_dtype, (d,))]))
    rec["d"] = d
    rec["v"] = mat
    Path(path).write_bytes(rec.tobytes() if n else b"")


def write_fvecs(path, dataset) -> None:
    data = dataset.data if hasattr(dataset, "data") else np.asarray(dataset, dtype=np.float32)
    _write_records(path, np.asarray(data, dtype=np.float32), "<f4")


def read_ivecs(path) -> np.ndarray:
    """Integer matrix (ground-truth neighbour lists); negatives are rejected."""
    data = _records(path, np.dtype("<i4"), "ivecs")
    neg = data < 0
    if neg.any():
        row, col = divmod(int(np.flatnonzero(neg.ravel())[0]), data.shape[1])
        raise FormatError("negative index in ivecs payload", offset=row * (4 + data.shape[1] * 4) + 4 + col * 4)
    return data.astype(np.int32)


def write_ivecs(path, matrix) -> None:
    _write_records(path, np.asarray(matrix, dtype="<i4"), "<i4")


def read_bvecs(path) -> VectorDataset:
    """uint8 payload records, widened to float32 (io.py:100-104).  For the GPU
    path without the widening copy use ``encode_file``."""
    data = _records(path, np.dtype("u1"), "bvecs")
    return VectorDataset(data=data.astype(np.float32), source=str(path))


def write_bvecs(path, matrix) -> None:
    _write_records(path, np.asarray(matrix, dtype=np.uint8), "u1")


def synth_dataset(n: int, d: int, clusters: int, seed: int, noise: float = 0.05) -> VectorDataset:
    """Seeded Gaussian mixture: means U[-1, 1]^d, isotropic noise (io.py:124-137;
    the same PCG64 draws in the same order, so the same bits)."""
    if n < 1 or d < 1 or clusters < 1:
        raise ConfigError("n, d, clusters must all be >= 1")
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.uniform(-1.0, 1.0, size=(clusters, d)).astype(np.float32)
    labels = rng.integers(0, clusters, size=n)
    data = means[labels] + rng.normal(0.0, noise, size=(n, d)).astype(np.float32)
    return VectorDataset(data=np.ascontiguousarray(data, dtype=np.float32),
                         source=f"synth(n={n},d={d},clusters={clusters},seed={seed},noise={noise})")


# ---------------------------------------------------------------- containers

def _checked_payload(raw: bytes, path) -> bytes:
    """Strip and verify the trailing CRC-32 (io.py:140-151)."""
    if len(raw) < 4:
        raise FormatError(f"file too short for checksum: {path}", offset=len(raw))
    payload = raw[:-4]
    if zlib.crc32(payload) != struct.unpack("<I", raw[-4:])[0]:
        raise FormatError(f"checksum mismatch in {path}", offset=len(payload))
    return payload


def write_codebooks(path, codebooks) -> None:
    cbs = list(codebooks)
    if not cbs:
        raise ConfigError("no codebooks to write")
    k, sub = cbs[0].k, cbs[0].sub_dim
    if any(cb.k != k or cb.sub_dim != sub for cb in cbs):
        raise ConfigError("codebooks disagree on sub_dim or k")
    m = len(cbs)
    payload = b"".join([_CODEBOOK_HEADER.pack(FORMAT_VERSION, m * sub, m, sub, k)]
                       + [cb.centroids_rowmajor.astype("<f4").tobytes() for cb in cbs]
                       + [cb.biases.astype("<f4").tobytes() for cb in cbs])
    Path(path).write_bytes(CODEBOOK_MAGIC + payload + struct.pack("<I", zlib.crc32(payload)))


def read_codebooks(path) -> list[Codebook]:
    raw = Path(path).read_bytes()
    if raw[:4] != CODEBOOK_MAGIC:
        raise FormatError(f"bad codebook magic in {path}", offset=0)
    payload = _checked_payload(raw[4:], path)
    if len(payload) < _CODEBOOK_HEADER.size:
        raise FormatError(f"truncated codebook header in {path}", offset=4)
    version, d, m, sub, k = _CODEBOOK_HEADER.unpack_from(payload, 0)
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported codebook version {version}", offset=4)
    if d != m * sub:
        raise FormatError(f"inconsistent dims d={d}, m={m}, sub_dim={sub}", offset=8)
    need = _CODEBOOK_HEADER.size + m * k * sub * 4 + m * k * 4
    if len(payload) != need:
        raise FormatError(f"codebook payload size {len(payload)} != expected {need}", offset=20)
    cents = np.frombuffer(payload, dtype="<f4", count=m * k * sub, offset=20).reshape(m, k, sub)
    biases = np.frombuffer(payload, dtype="<f4", count=m * k, offset=20 + m * k * sub * 4).reshape(m, k)
    out = []
    for j in range(m):
        cb = Codebook.from_rowmajor(j, cents[j])
        out.append(Codebook(j, cb.centroids_rowmajor, cb.centroids_transposed,
                            _readonly(np.array(biases[j], dtype=np.float32))))
    return out


def _codes_header(n: int, m: int, k: int) -> bytes:
    return _CODES_HEADER.pack(FORMAT_VERSION, n, m, k, 1 if k <= 256 else 2)


def write_codes(path, codes, k: int | None = None) -> None:
    """PQCD file from a PQCodes (host) or, with ``k``, from a CUDA tensor of
    codes -- then the CRC-32 is computed on the GPU (cspq_crc32_device) and
    only the codes themselves cross PCIe."""
    if isinstance(codes, PQCodes):
        arr = codes.codes.astype("<u1" if codes.k <= 256 else "<u2")
        header = _codes_header(codes.n, codes.m, codes.k)
        payload = header + arr.tobytes()
        Path(path).write_bytes(CODES_MAGIC + payload + struct.pack("<I", zlib.crc32(payload)))
        return
    from ._device import torch
    t = torch()
    if not (isinstance(codes, t.Tensor) and codes.is_cuda) or k is None:
        raise ConfigError("write_codes takes a PQCodes, or a CUDA codes tensor together with k")
    want = t.uint8 if k <= 256 else t.uint16
    if codes.dtype != want or codes.dim() != 2:
        raise ConfigError(f"codes tensor must be 2-D {want} for k={k}")
    c = codes.contiguous()
    n, m = c.shape
    header = _codes_header(n, m, k)
    crc = crc32_device(c, zlib.crc32(header))
    with open(path, "wb") as f:
        f.write(CODES_MAGIC + header)
        f.write(c.cpu().numpy().tobytes())
        f.write(struct.pack("<I", crc))


def read_codes(path) -> PQCodes:
    raw = Path(path).read_bytes()
    if raw[:4] != CODES_MAGIC:
        raise FormatError(f"bad codes magic in {path}", offset=0)
    payload = _checked_payload(raw[4:], path)
    if len(payload) < _CODES_HEADER.size:
        raise FormatError(f"truncated codes header in {path}", offset=4)
    version, n, m, k, width = _CODES_HEADER.unpack_from(payload, 0)
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported codes version {version}", offset=4)
    if width not in (1, 2) or (width == 1) != (k <= 256):
        raise FormatError(f"invalid code width {width} for k={k}", offset=20)
    need = _CODES_HEADER.size + n * m * width
    if len(payload) != need:
        raise FormatError(f"codes payload size {len(payload)} != expected {need}", offset=24)
    arr = np.frombuffer(payload, dtype="<u1" if width == 1 else "<u2", count=n * m, offset=24)
    return PQCodes(codes=np.array(arr.reshape(n, m), dtype=np.uint8 if width == 1 else np.uint16), k=k)


# ---------------------------------------------------------------- GPU paths

def crc32_device(data, crc_in: int = 0) -> int:
    """zlib.crc32(bytes(data), crc_in) of a CUDA tensor, computed on the GPU."""
    from ._device import ptr, stream_ptr, torch
    t = torch()
    N.require_cuda()
    if not (isinstance(data, t.Tensor) and data.is_cuda):
        raise ConfigError("crc32_device needs a CUDA tensor")
    c = data.contiguous()
    nbytes = c.numel() * c.element_size()
    ws = t.empty(N.load().cspq_crc32_workspace_bytes(nbytes), dtype=t.uint8, device=c.device)
    out = t.empty(1, dtype=t.int32, device=c.device)
    N.call("cspq_crc32_device", ptr(c), nbytes, int(crc_in) & 0xFFFFFFFF, ptr(out), ptr(ws), stream_ptr(c.device))
    return int(out.cpu().numpy().view(np.uint32)[0])


_FILE_ERRORS = {
    1: lambda kind, off, v, path: FormatError(f"empty dataset: {path}", offset=0),
    2: lambda kind, off, v, path: FormatError(f"truncated {kind} record header", offset=off),
    3: lambda kind, off, v, path: FormatError(f"non-positive {kind} record length {v}", offset=off),
    4: None,  # needs the first record length
    5: lambda kind, off, v, path: FormatError(f"truncated {kind} record body", offset=off),
    6: lambda kind, off, v, path: FormatError(f"non-finite value in {kind} payload", offset=off),
}


def encode_file(in_path, codebooks, out_path, plan=None, *, precomputed_bias: bool = True,
                fmt: str | None = None) -> dict:
    """Stream an fvecs / bvecs file into a PQCD codes file on the GPU
    (cspq_encode_vecs_file): the equivalent of
    ``write_codes(out, encode_dataset(read_fvecs(in), codebooks))`` with the
    same codes, the same file bytes and the same FormatErrors, without holding
    the dataset in memory.  Returns {"n", "m", "k"}."""
    from .bulk import CodebookSet, EncoderVariant, ExecutionPlan, _MODES, _variant_args
    from ._device import device as _device, ptr, torch
    N.require_cuda()
    plan = plan or ExecutionPlan()
    fmt = fmt or Path(in_path).suffix.lstrip(".").lower()
    if fmt not in ("fvecs", "bvecs"):
        raise ConfigError(f"unknown vector file format {fmt!r} (fvecs or bvecs)")
    cbset = CodebookSet.from_codebooks(codebooks)
    head = np.fromfile(in_path, dtype="<i4", count=1)
    if head.shape[0] == 1 and int(head[0]) > 0 and int(head[0]) != cbset.d:
        # the reference reads (and rejects malformed files) before encode_dataset checks d
        (read_fvecs if fmt == "fvecs" else read_bvecs)(in_path)
        raise ConfigError(f"dataset dimensionality {int(head[0])} does not match codebooks' d={cbset.d}")
    dev = _device(plan.device)
    rm, bs, guard, vid = _variant_args(cbset, plan, precomputed_bias, dev)
    img = None
    if plan.mode in ("auto", "tensor") and vid != N.VARIANT_REFERENCE and cbset.k == 256 and cbset.sub_dim in (4, 8):
        img = cbset.tc_image(dev, nobias=not precomputed_bias and plan.variant is EncoderVariant.BLOCKED)
    elif plan.mode == "tensor":
        raise ConfigError("mode='tensor' needs k=256, sub_dim in {4, 8} and a REFORMULATED/BLOCKED variant")
    torch().cuda.current_stream(dev).synchronize()  # codebook tables visible to the pipeline's streams
    nrows = ctypes.c_int64(0)
    err = (ctypes.c_int64 * 3)()
    rc = N.load().cspq_encode_vecs_file(
        os.fsencode(str(in_path)), 0 if fmt == "fvecs" else 1, os.fsencode(str(out_path)), ptr(rm), ptr(bs),
        ptr(guard), ptr(img), cbset.m, cbset.k, cbset.sub_dim, vid, _MODES[plan.mode],
        plan.resolved_batch_rows(cbset.d * (4 if fmt == "fvecs" else 1)), min(plan.streams, 8), dev.index, ctypes.byref(nrows), err)
    if rc == N.CSPQ_E_FORMAT:
        kind, off, val = int(err[0]), int(err[1]), int(err[2])
        if kind == 4:
            first = int(np.fromfile(in_path, dtype="<i4", count=1)[0])
            raise FormatError(f"inconsistent {fmt} record length {val} (expected {first})", offset=off)
        raise _FILE_ERRORS[kind](fmt, off, val, in_path)
    if rc != N.CSPQ_OK:
        N.raise_status(rc, "cspq_encode_vecs_file")
    return {"n": int(nrows.value), "m": cbset.m, "k": cbset.k}
