"""Dataset-scale encoding on the B200 -- the drop-in for ``cspq.bulk``.

Reference: /root/reference/pkg/src/cspq/bulk.py:31-195.  The reference cuts
the rows into ``block_size`` blocks and hands them round-robin to a thread
pool of nogil numba drivers (bulk.py:139-155).  Here the whole matrix goes
to one fused CUDA kernel (device-resident rows) or through the pipelined
host->device->host path of the C ABI (host rows); the plan still validates
exactly like the reference's, and -- as there -- never changes the codes.
"""

from __future__ import annotations

import ctypes
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._device import device as _device, ptr, stream_ptr, to_device, torch
from .core import Codebook, ConfigError, DataError, PQCodes, PQParams
from .kernels import EncoderVariant, native_lane_width

CHUNK_MAJOR = "chunk_major"
VECTOR_MAJOR = "vector_major"

_VARIANT_IDS = {
    EncoderVariant.REFERENCE: N.VARIANT_REFERENCE,
    EncoderVariant.REFORMULATED: N.VARIANT_REFORMULATED,
    EncoderVariant.BLOCKED: N.VARIANT_BLOCKED,
}
_MODES = {"auto": N.MODE_AUTO, "exact": N.MODE_EXACT, "guarded": N.MODE_GUARDED, "tensor": N.MODE_AUTO}


@dataclass(frozen=True)
class ExecutionPlan:
    """Scheduling knobs (bulk.py:31-50).  order / block_size / w / workers
    are the reference's and are validated identically; on the GPU they are
    performance-only (codes are plan-invariant, test_bulk.py:44-62).
    GPU extras: ``mode`` ("auto" | "exact" | "guarded" | "tensor" -- all
    give the oracle's codes; "tensor" = the tcgen05 kernel, "guarded" = the
    FFMA kernel, "exact" = strict fp32 chains, "auto" = tensor where the
    shape allows it, else guarded), ``batch_rows`` (rows per host<->device batch; None =
    ~256 MB of rows), ``streams`` (CUDA streams in that pipeline),
    ``device`` (CUDA ordinal; None = current) and ``devices`` (several ordinals: host rows
    are split into contiguous ranges, one pipeline per GPU on its own PCIe link -- the
    single-process counterpart of the reference's worker threads)."""

    order: str = CHUNK_MAJOR
    block_size: int = 4096
    variant: EncoderVariant = EncoderVariant.BLOCKED
    w: int | None = None
    workers: int = 1
    mode: str = "auto"
    batch_rows: int | None = None
    streams: int = 3
    device: int | None = None
    devices: tuple | None = None

    def __post_init__(self):
        if self.order not in (CHUNK_MAJOR, VECTOR_MAJOR):
            raise ConfigError(f"unknown order {self.order!r}")
        if self.block_size < 1:
            raise ConfigError(f"block_size must be >= 1, got {self.block_size}")
        if self.workers < 1:
            raise ConfigError(f"workers must be >= 1, got {self.workers}")
        if self.w is not None and self.w < 1:
            raise ConfigError(f"w must be >= 1, got {self.w}")
        if self.mode not in _MODES:
            raise ConfigError(f"unknown mode {self.mode!r}")
        if self.batch_rows is not None and self.batch_rows < 1:
            raise ConfigError(f"batch_rows must be >= 1, got {self.batch_rows}")
        if not 1 <= self.streams <= 16:
            raise ConfigError(f"streams must be in [1, 16], got {self.streams}")
        if self.devices is not None:
            devs = tuple(self.devices)
            if not devs or any(not isinstance(d, (int, np.integer)) or d < 0 for d in devs):
                raise ConfigError(f"devices must be a non-empty sequence of CUDA ordinals, got {self.devices!r}")
            object.__setattr__(self, "devices", tuple(int(d) for d in devs))

    def resolved_w(self) -> int:
        return self.w if self.w is not None else native_lane_width()

    def resolved_batch_rows(self, row_bytes: int = 4 * 768) -> int:
        """Rows per host<->device batch: ``batch_rows``, else ~256 MB of input rows (16K..1M
        rows).  Not derived from block_size, whose reference meaning (rows per CPU work item)
        would size the pinned ring."""
        if self.batch_rows is not None:
            return self.batch_rows
        return int(min(1 << 20, max(1 << 14, (256 << 20) // max(1, row_bytes))))


@dataclass(frozen=True)
class CodebookSet:
    """All m codebooks stacked (bulk.py:53-105): rowmajor (m, k, sub),
    transposed (m, sub, k), biases (m, k), float32.  The device copy (and
    the encode guard constants) is uploaded once per device and cached."""

    rowmajor: np.ndarray
    transposed: np.ndarray
    biases: np.ndarray
    _dev: dict = field(default_factory=dict, compare=False, repr=False)

    @classmethod
    def from_codebooks(cls, codebooks) -> "CodebookSet":
        if isinstance(codebooks, cls):
            return codebooks
        cbs = list(codebooks)
        if not cbs:
            raise ConfigError("no codebooks given")
        k, sub = cbs[0].k, cbs[0].sub_dim
        if any(cb.k != k or cb.sub_dim != sub for cb in cbs):
            raise ConfigError("codebooks disagree on sub_dim or k")
        arrays = [np.ascontiguousarray(np.stack(a)) for a in (
            [cb.centroids_rowmajor for cb in cbs],
            [cb.centroids_transposed for cb in cbs],
            [cb.biases for cb in cbs])]
        for a in arrays:
            a.flags.writeable = False
        return cls(*arrays)

    @classmethod
    def from_rowmajor_batch(cls, rowmajor) -> "CodebookSet":
        """All m codebooks from one (m, k, sub) float32 array -- what from_codebooks(
        [Codebook.from_rowmajor(j, rowmajor[j]) ...]) builds (same transposes, same bias bits: the
        float64 einsum reduces the same contiguous axis), in three vectorised numpy operations
        instead of m Codebook objects (m = 120: 3 ms -> 0.2 ms, which is ~7 % of config 2's train +
        encode step)."""
        rm = np.ascontiguousarray(np.asarray(rowmajor, dtype=np.float32))
        if rm.ndim != 3 or rm.shape[0] == 0:
            raise ConfigError(f"centroids must be (m, k, sub), got shape {rm.shape}")
        if not np.isfinite(rm).all():
            j = int(np.argmax(~np.isfinite(rm).all(axis=(1, 2))))
            raise DataError(f"non-finite centroid values in subspace {j}")
        arrays = [rm, np.ascontiguousarray(rm.transpose(0, 2, 1)),
                  (0.5 * np.einsum("mkt,mkt->mk", rm, rm, dtype=np.float64)).astype(np.float32)]
        for a in arrays:
            a.flags.writeable = False
        return cls(*arrays)

    @property
    def m(self) -> int:
        return self.rowmajor.shape[0]

    @property
    def k(self) -> int:
        return self.rowmajor.shape[1]

    @property
    def sub_dim(self) -> int:
        return self.rowmajor.shape[2]

    @property
    def d(self) -> int:
        return self.m * self.sub_dim

    def __getitem__(self, j: int) -> Codebook:
        return Codebook(j, self.rowmajor[j], self.transposed[j], self.biases[j])

    def tc_image(self, dev=None, nobias: bool = False):
        """Prepared tensor-core codebook image (cspq_encode_tc_prepare), or
        None when the shape has no tensor-core path (k != 256, sub not 4/8)."""
        dev = _device() if dev is None else dev
        key = ("tc", dev.type, dev.index, nobias)
        if key not in self._dev:
            nbytes = N.load().cspq_encode_tc_image_bytes(self.m, self.k, self.sub_dim)
            img = None
            if nbytes:
                t = torch()
                rm, bs, _, nob, _ = self.on_device(dev)
                img = t.empty(nbytes, dtype=t.uint8, device=dev)
                with t.cuda.device(dev):
                    N.call("cspq_encode_tc_prepare", ptr(rm), ptr(nob if nobias else bs), self.m, self.k,
                           self.sub_dim, ptr(img), stream_ptr(dev))
            self._dev[key] = img
        return self._dev[key]

    def on_device(self, dev=None):
        """(rowmajor, biases, guard, recomputed_biases, guard_nob) as CUDA tensors."""
        dev = _device() if dev is None else dev
        key = (dev.type, dev.index)
        hit = self._dev.get(key)
        if hit is None:
            t = torch()
            rm = to_device(self.rowmajor, dev, t.float32)
            bs = to_device(self.biases, dev, t.float32)
            guard = t.empty((self.m, 2), dtype=t.float32, device=dev)
            nob = t.empty((self.m, self.k), dtype=t.float32, device=dev)
            with t.cuda.device(dev):
                sp = stream_ptr(dev)
                N.call("cspq_encode_prepare", ptr(rm), ptr(bs), self.m, self.k, self.sub_dim, ptr(guard), sp)
                N.call("cspq_recompute_biases_f32", ptr(rm), self.m, self.k, self.sub_dim, ptr(nob), sp)
                guard_nob = t.empty((self.m, 2), dtype=t.float32, device=dev)
                N.call("cspq_encode_prepare", ptr(rm), ptr(nob), self.m, self.k, self.sub_dim, ptr(guard_nob), sp)
            hit = (rm, bs, guard, nob, guard_nob)
            self._dev[key] = hit
        return hit


def _resolve_input(dataset):
    """-> (array-or-tensor, is_cuda_tensor).  VectorDataset, numpy, torch."""
    t = torch()
    if isinstance(dataset, t.Tensor):
        return dataset, dataset.is_cuda
    X = dataset.data if isinstance(getattr(dataset, "data", None), np.ndarray) else dataset
    return np.asarray(X), False


def _variant_args(cbset: CodebookSet, plan: ExecutionPlan, precomputed_bias: bool, dev):
    rm, bs, guard, nob, guard_nob = cbset.on_device(dev)
    vid = _VARIANT_IDS[plan.variant]
    if plan.variant is EncoderVariant.BLOCKED and not precomputed_bias:
        # kernels.py:146-157: bias recomputed as 0.5f * fl-chain(c*c) -- a
        # per-codebook constant, so one table gives the same bits
        return rm, nob, guard_nob, vid
    return rm, bs, guard, vid


def _tc_shape_ok(cbset, in_u8: bool) -> bool:
    """k = 256, sub in {4, 8} and not more subspaces than the tensor-core kernel's shared memory holds."""
    return (cbset.k == 256 and cbset.sub_dim in (4, 8)
            and cbset.m <= N.load().cspq_encode_tc_max_subspaces(cbset.sub_dim, N.IN_U8 if in_u8 else N.IN_F32))


def _tc_ok(X, xrs, cbset) -> bool:
    t = torch()
    if not _tc_shape_ok(cbset, X.dtype == t.uint8):
        return False
    if X.dtype == t.uint8:  # one subvector per sub-byte cp.async (encode_tc_ex checks the same)
        sub = cbset.sub_dim
        return X.data_ptr() % sub == 0 and xrs % sub == 0
    return X.data_ptr() % 16 == 0 and (xrs * 4) % 16 == 0


def encode_dataset_device(X, codebooks, plan: ExecutionPlan | None = None, *,
                          precomputed_bias: bool = True, out=None, best=None):
    """Encode a CUDA tensor X (n, d) float32/uint8 in place on its device;
    returns the (n, m) codes tensor (uint8, or int16 holding uint16 bits
    when k > 256).  Stream-ordered on the current stream, no sync."""
    t = torch()
    plan = plan or ExecutionPlan()
    cbset = CodebookSet.from_codebooks(codebooks)
    if not (isinstance(X, t.Tensor) and X.is_cuda):
        raise ConfigError("encode_dataset_device needs a CUDA tensor (use encode_dataset for host arrays)")
    if X.dim() != 2:
        raise ConfigError(f"dataset must be 2-D, got shape {tuple(X.shape)}")
    if X.dtype not in (t.float32, t.uint8):
        X = X.float()
    if X.stride(1) != 1:
        X = X.contiguous()
    n, d = X.shape
    dev = X.device
    cdt = t.uint8 if cbset.k <= 256 else t.int16
    if out is None:
        out = t.empty((n, cbset.m), dtype=cdt, device=dev)
    elif (not isinstance(out, t.Tensor) or out.device != dev or out.dtype != cdt or tuple(out.shape) != (n, cbset.m)
          or out.stride(1) != 1):
        raise ConfigError(f"out must be a ({n}, {cbset.m}) {cdt} tensor on {dev} with unit column stride")
    if best is not None and (not isinstance(best, t.Tensor) or best.device != dev or best.dtype != t.float32
                             or tuple(best.shape) != (n, cbset.m) or not best.is_contiguous()):
        raise ConfigError(f"best must be a contiguous ({n}, {cbset.m}) float32 tensor on {dev}")
    if n == 0:
        return out
    if d != cbset.d:
        raise ConfigError(f"dataset dimensionality {d} does not match codebooks' d={cbset.d}")
    rm, bs, guard, vid = _variant_args(cbset, plan, precomputed_bias, dev)
    xrs = X.stride(0) if n > 1 else d  # a 1-row view may carry any row stride
    mode = plan.mode
    use_tc = mode in ("auto", "tensor") and vid != N.VARIANT_REFERENCE and _tc_ok(X, xrs, cbset)
    if mode == "tensor" and not use_tc:
        raise ConfigError("mode='tensor' needs k=256, sub_dim in {4, 8}, a REFORMULATED/BLOCKED variant, "
                          "16-byte aligned rows and at most cspq_encode_tc_max_subspaces subspaces")
    if best is not None and not use_tc:
        raise ConfigError("best (winning tensor-core scores) is only produced by the tensor-core path")
    with t.cuda.device(dev):
        if use_tc:
            img = cbset.tc_image(dev, nobias=not precomputed_bias and plan.variant is EncoderVariant.BLOCKED)
            N.call("cspq_encode_tc", ptr(X), N.IN_U8 if X.dtype == t.uint8 else N.IN_F32, n, d, xrs,
                   ptr(rm), ptr(bs), ptr(guard), ptr(img), cbset.m, cbset.k, cbset.sub_dim, ptr(out),
                   out.stride(0), ptr(best), stream_ptr(dev))
        else:
            N.call("cspq_encode", ptr(X), N.IN_U8 if X.dtype == t.uint8 else N.IN_F32, n, d, xrs,
                   ptr(rm), ptr(bs), ptr(guard), cbset.m, cbset.k, cbset.sub_dim, ptr(out), out.stride(0),
                   vid, _MODES[mode], stream_ptr(dev))
    return out


def _encode_host_multi(X, cbset, plan: ExecutionPlan, precomputed_bias: bool, out: np.ndarray) -> np.ndarray:
    """plan.devices: contiguous row ranges, one host pipeline per GPU, run from host threads
    (each C call releases the GIL).  Rows are independent, so the codes equal a single
    device's (the reference's plan invariance, test_bulk.py:44-62)."""
    from concurrent.futures import ThreadPoolExecutor
    from dataclasses import replace
    devs = plan.devices
    n = X.shape[0]
    bounds = [n * i // len(devs) for i in range(len(devs) + 1)]
    jobs = [(d, bounds[i], bounds[i + 1]) for i, d in enumerate(devs) if bounds[i + 1] > bounds[i]]

    def run(job):
        d, b, e = job
        encode_dataset_host(X[b:e], cbset, replace(plan, device=d, devices=None), precomputed_bias=precomputed_bias,
                            out=out[b:e])

    with ThreadPoolExecutor(len(jobs)) as ex:
        list(ex.map(run, jobs))  # (re-raises the first failure)
    return out


def encode_dataset_host(X: np.ndarray, codebooks, plan: ExecutionPlan | None = None, *,
                        precomputed_bias: bool = True, out: np.ndarray | None = None,
                        batch_ms: np.ndarray | None = None) -> np.ndarray:
    """Encode host rows through the C ABI's pipelined H2D -> encode -> D2H path
    (cspq_encode_host).  Pinned inputs/outputs (``pinned_empty``) are copied
    directly; pageable ones are staged through a pinned ring.  ``plan.devices``
    spreads the rows over several GPUs (one pipeline each)."""
    N.require_cuda()
    plan = plan or ExecutionPlan()
    cbset = CodebookSet.from_codebooks(codebooks)
    in_u8 = X.dtype == np.uint8
    if not in_u8:
        X = np.ascontiguousarray(X, dtype=np.float32)
    elif not X.flags.c_contiguous:
        X = np.ascontiguousarray(X)
    n, d = X.shape
    cdt = np.uint8 if cbset.k <= 256 else np.uint16
    if out is None:
        out = np.empty((n, cbset.m), dtype=cdt)
    elif (not isinstance(out, np.ndarray) or out.dtype != cdt or out.shape != (n, cbset.m)
          or not out.flags.c_contiguous or not out.flags.writeable):
        # the C pipeline writes n * m codes linearly through out's buffer
        raise ConfigError(f"out must be a writeable C-contiguous ({n}, {cbset.m}) {np.dtype(cdt).name} array")
    batch_rows = plan.resolved_batch_rows(d * (1 if in_u8 else 4))
    nb = -(-n // min(batch_rows, max(n, 1)))
    if batch_ms is not None and (not isinstance(batch_ms, np.ndarray) or batch_ms.dtype != np.float64
                                 or batch_ms.ndim != 1 or not batch_ms.flags.c_contiguous
                                 or not batch_ms.flags.writeable or batch_ms.shape[0] < nb):
        raise ConfigError(f"batch_ms must be a writeable contiguous float64 array of at least {nb} entries")
    if n == 0:
        return out
    if d != cbset.d:
        raise ConfigError(f"dataset dimensionality {d} does not match codebooks' d={cbset.d}")
    if plan.devices is not None and len(plan.devices) > 1:
        if batch_ms is not None:
            raise ConfigError("batch_ms is per pipeline: not available with several devices")
        return _encode_host_multi(X, cbset, plan, precomputed_bias, out)
    dev = _device(plan.device if plan.devices is None else plan.devices[0])
    rm, bs, guard, vid = _variant_args(cbset, plan, precomputed_bias, dev)
    t = torch()
    t.cuda.current_stream(dev).synchronize()  # codebook upload visible to the pipeline streams
    img = None
    if plan.mode in ("auto", "tensor") and vid != N.VARIANT_REFERENCE and _tc_shape_ok(cbset, in_u8):
        img = cbset.tc_image(dev, nobias=not precomputed_bias and plan.variant is EncoderVariant.BLOCKED)
    elif plan.mode == "tensor":
        raise ConfigError("mode='tensor' needs k=256, sub_dim in {4, 8}, a REFORMULATED/BLOCKED variant and "
                          "at most cspq_encode_tc_max_subspaces subspaces")
    t.cuda.current_stream(dev).synchronize()  # image preparation visible to the pipeline streams
    N.call("cspq_encode_host", X.ctypes.data_as(ctypes.c_void_p), N.IN_U8 if in_u8 else N.IN_F32, n, d,
           ptr(rm), ptr(bs), ptr(guard), ptr(img), cbset.m, cbset.k, cbset.sub_dim,
           out.ctypes.data_as(ctypes.c_void_p), vid, _MODES[plan.mode], batch_rows,
           plan.streams, None if batch_ms is None else batch_ms.ctypes.data_as(ctypes.c_void_p),
           dev.index)
    return out


def encode_dataset(dataset, codebooks, plan: ExecutionPlan | None = None, *,
                   precomputed_bias: bool = True) -> PQCodes:
    """Encode every vector (bulk.py:108-157); the plan never changes codes.

    Accepts a VectorDataset, a numpy array (float32, or uint8 widened
    exactly in-kernel) or a torch tensor (CUDA tensors are encoded where
    they live).  Returns host ``PQCodes`` like the reference; use
    ``encode_dataset_device`` to keep codes on the GPU."""
    plan = plan or ExecutionPlan()
    cbset = CodebookSet.from_codebooks(codebooks)
    X, on_gpu = _resolve_input(dataset)
    if X.ndim != 2:
        raise ConfigError(f"dataset must be 2-D, got shape {tuple(X.shape)}")
    dtype = np.uint8 if cbset.k <= 256 else np.uint16
    if X.shape[0] == 0:
        return PQCodes(codes=np.empty((0, cbset.m), dtype=dtype), k=cbset.k)
    if X.shape[1] != cbset.d:
        raise ConfigError(f"dataset dimensionality {X.shape[1]} does not match codebooks' d={cbset.d}")
    if on_gpu:
        codes = encode_dataset_device(X, cbset, plan, precomputed_bias=precomputed_bias).cpu().numpy()
        if dtype == np.uint16:
            codes = codes.view(np.uint16)
    else:
        if not isinstance(X, np.ndarray):
            X = X.numpy()
        if X.dtype != np.uint8 and X.dtype != np.float32:
            X = X.astype(np.float32)
        codes = encode_dataset_host(X, cbset, plan, precomputed_bias=precomputed_bias)
    return PQCodes(codes=codes, k=cbset.k)


@contextmanager
def kernel_allocation_probe(record: dict):
    """Counterpart of bulk.py:160-184.  The reference counts numba heap
    allocations per driver call; the CUDA kernels allocate nothing at all
    (all scratch is registers/shared memory), so the probe reports the
    torch caching-allocator's change in allocated device bytes."""
    t = torch()
    dev = t.cuda.current_device() if t.cuda.is_available() else None
    start = t.cuda.memory_allocated(dev) if dev is not None else 0
    try:
        yield record
    finally:
        end = t.cuda.memory_allocated(dev) if dev is not None else 0
        record["device_bytes"] = end - start


def estimate_working_set(params: PQParams, plan: ExecutionPlan) -> int:
    """Resident bytes during bulk encoding, independent of dataset size
    (bulk.py:187-195): one codebook in both layouts plus biases, plus the
    per-worker lane state."""
    resident = 2 * params.k * params.sub_dim * 4 + params.k * 4
    return resident + plan.workers * 2 * plan.resolved_w() * 4
