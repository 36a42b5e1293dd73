"""Per-subvector encoder API -- the drop-in for ``cspq.kernels``' public
functions (/root/reference/pkg/src/cspq/kernels.py:36-81, 340-441).

Every call runs on the GPU through ``cspq_encode_with_scores`` (the exact
kernel: strict fp32 chains, first index on ties), so the returned
(code, score) pairs carry the oracle's bits.  The three variants keep the
reference's semantics:

* REFERENCE    -- argmin (||v||^2 + ||c||^2) - 2<v,c>      (kernels.py:84-105)
* REFORMULATED -- argmin b - <v,c>, b = 0.5||c||^2          (kernels.py:108-122)
* BLOCKED      -- same scores as REFORMULATED for every lane
                  width w (kernels.py:125-168); w is validated and then
                  only a CPU scheduling notion, so it cannot change a bit.
"""

from __future__ import annotations

import enum

import numpy as np

from .core import Codebook, ConfigError, Error, ScoreBlock

__all__ = [
    "EncoderVariant", "native_lane_width", "encode_ref", "encode_ref_with_score",
    "encode_reform", "encode_reform_with_score", "encode_blocked", "encode_blocked_with_score",
    "encode_vector",
]


class EncoderVariant(enum.Enum):
    REFERENCE = "reference"
    REFORMULATED = "reformulated"
    BLOCKED = "blocked"


def native_lane_width() -> int:
    """Host float32 SIMD width (kernels.py:61-81): 16 with AVX-512, 8 with
    AVX/AVX2, else 4; 8 when /proc/cpuinfo is unreadable.  Kept for API
    parity -- the GPU kernels do not depend on it."""
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((ln for ln in f if ln.startswith("flags")), "")
    except OSError:
        return 8
    if "avx512f" in flags:
        return 16
    if "avx" in flags:
        return 8
    return 4 if flags else 8


def _subvector(v, cb: Codebook) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(v, dtype=np.float32))
    if arr.ndim != 1 or arr.shape[0] != cb.sub_dim:
        raise ConfigError(f"subvector length {arr.shape} does not match sub_dim={cb.sub_dim}")
    return arr


def _gpu_one(arr: np.ndarray, rowmajor: np.ndarray, biases, variant_id: int):
    from . import _native as N
    from ._device import device, ptr, stream_ptr, to_device, torch
    t = torch()
    dev = device()
    k, sub = rowmajor.shape
    x = to_device(arr.reshape(1, sub), dev, t.float32)
    cb = to_device(np.ascontiguousarray(rowmajor, dtype=np.float32).reshape(1, k, sub), dev, t.float32)
    b = to_device(np.ascontiguousarray(biases, dtype=np.float32).reshape(1, k), dev, t.float32) \
        if biases is not None else cb  # REFERENCE never reads B
    codes = t.empty((1, 1), dtype=t.int32, device=dev)
    best = t.empty((1, 1), dtype=t.float32, device=dev)
    N.call("cspq_encode_with_scores", ptr(x), N.IN_F32, 1, sub, sub, ptr(cb), ptr(b), 1, k, sub,
           ptr(codes), ptr(best), variant_id, stream_ptr(dev))
    return int(codes.item()), np.float32(best.item())


def encode_ref(v, cb: Codebook) -> int:
    """Nearest centroid by the fully expanded squared distance."""
    return encode_ref_with_score(v, cb)[0]


def encode_ref_with_score(v, cb: Codebook) -> tuple[int, np.float32]:
    from ._native import VARIANT_REFERENCE
    return _gpu_one(_subvector(v, cb), cb.centroids_rowmajor, None, VARIANT_REFERENCE)


def encode_reform(v, cb: Codebook) -> int:
    """Nearest centroid by bias - <v, c>."""
    return encode_reform_with_score(v, cb)[0]


def encode_reform_with_score(v, cb: Codebook) -> tuple[int, np.float32]:
    from ._native import VARIANT_REFORMULATED
    arr = _subvector(v, cb)
    if cb.biases is None or cb.biases.shape[0] != cb.k:
        raise ConfigError("codebook biases not populated")
    return _gpu_one(arr, cb.centroids_rowmajor, cb.biases, VARIANT_REFORMULATED)


def encode_blocked(v, cb: Codebook, w: int | None = None) -> int:
    """Nearest centroid, w centroids per block (identical codes for any w)."""
    return encode_blocked_with_score(v, cb, w)[0]


def encode_blocked_with_score(v, cb: Codebook, w: int | None = None) -> tuple[int, np.float32]:
    from ._native import VARIANT_BLOCKED
    arr = _subvector(v, cb)
    ct = cb.centroids_transposed
    if ct is None or ct.shape != (cb.sub_dim, cb.k):
        raise ConfigError("codebook transposed layout not populated")
    w = native_lane_width() if w is None else w
    if w < 1:
        raise ConfigError(f"w must be >= 1, got {w}")
    sb = ScoreBlock(w)
    # the GPU reads the dimension-major layout back as row-major centroids
    sb.best_idx, sb.best_score = _gpu_one(arr, np.ascontiguousarray(ct.T), cb.biases, VARIANT_BLOCKED)
    return sb.best_idx, sb.best_score


def encode_vector(v, codebooks, variant: EncoderVariant = EncoderVariant.BLOCKED,
                  w: int | None = None) -> np.ndarray:
    """All m codes of one vector (chunk j through codebook j), uint8 for
    k <= 256 else uint16 (kernels.py:407-441)."""
    cbs = list(codebooks)
    if not cbs:
        raise ConfigError("no codebooks given")
    sub, k = cbs[0].sub_dim, cbs[0].k
    if any(cb.sub_dim != sub or cb.k != k for cb in cbs):
        raise ConfigError("codebooks disagree on sub_dim or k")
    arr = np.ascontiguousarray(np.asarray(v, dtype=np.float32))
    if arr.ndim != 1 or arr.shape[0] != sub * len(cbs):
        raise ConfigError(f"vector length {arr.shape} does not match d={sub * len(cbs)}")
    fn = {EncoderVariant.REFERENCE: lambda c, cb: encode_ref(c, cb),
          EncoderVariant.REFORMULATED: lambda c, cb: encode_reform(c, cb),
          EncoderVariant.BLOCKED: lambda c, cb: encode_blocked(c, cb, w)}[variant]
    out = np.empty(len(cbs), dtype=np.uint8 if k <= 256 else np.uint16)
    for j, cb in enumerate(cbs):
        try:
            out[j] = fn(arr[j * sub:(j + 1) * sub], cb)
        except Error as exc:
            raise type(exc)(f"chunk {j}: {exc}") from None
    return out
