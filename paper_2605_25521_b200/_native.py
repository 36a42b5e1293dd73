"""ctypes binding of the C ABI in include/cspq_b200.h.

The shared library ``_lib/libcspq_b200.so`` is built in-tree by
``csrc/Makefile`` (``__graft_entry__.build()``).  There is no fallback: if
the library is missing or CUDA is unavailable, every compute entry point
raises ``NativeUnavailable`` -- the product path never silently drops to a
CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# CSPQ_LIB_PATH: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("CSPQ_LIB_PATH") or os.path.join(HERE, "_lib", "libcspq_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "cspq_b200.h")

CSPQ_OK = 0
CSPQ_E_CONFIG = -1
CSPQ_E_DATA = -2
CSPQ_E_CUDA = -3
CSPQ_E_NOMEM = -4
CSPQ_E_TRAINING = -5
CSPQ_E_FORMAT = -6

IN_F32, IN_U8 = 0, 1
VARIANT_REFERENCE, VARIANT_REFORMULATED, VARIANT_BLOCKED = 0, 1, 2
MODE_AUTO, MODE_EXACT, MODE_GUARDED = 0, 1, 2

_i32, _i64, _vp, _dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
_SIGS = {
    "cspq_abi_version": ([], _i32),
    "cspq_last_error": ([], ctypes.c_char_p),
    "cspq_encode_stats": ([_vp, _i32], _i32),
    "cspq_launch_count": ([_i32], ctypes.c_uint64),
    "cspq_encode_set_tiling": ([_i32], _i32),
    "cspq_encode_tc_image_bytes": ([_i32, _i32, _i32], ctypes.c_size_t),
    "cspq_encode_tc_max_subspaces": ([_i32, _i32], _i32),
    "cspq_encode_tc_prepare": ([_vp, _vp, _i32, _i32, _i32, _vp, _vp], _i32),
    "cspq_encode_tc": ([_vp, _i32, _i64, _i32, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _vp, _vp], _i32),
    "cspq_encode_prepare": ([_vp, _vp, _i32, _i32, _i32, _vp, _vp], _i32),
    "cspq_recompute_biases_f32": ([_vp, _i32, _i32, _i32, _vp, _vp], _i32),
    "cspq_encode": ([_vp, _i32, _i64, _i32, _i64, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _i32, _i32, _vp], _i32),
    "cspq_encode_with_scores": ([_vp, _i32, _i64, _i32, _i64, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _i32, _vp], _i32),
    "cspq_encode_subspace_major": ([_vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp, _i32, _vp], _i32),
    "cspq_encode_host": ([_vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _i32, _i32, _i64, _i32, _vp, _i32], _i32),
    "cspq_lloyd_workspace_bytes": ([_i64, _i32, _i32, _i32], ctypes.c_size_t),
    "cspq_lloyd_assign": ([_vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp], _i32),
    "cspq_lloyd_accumulate": ([_vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_lloyd_update": ([_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_lloyd_repair": ([_vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_lloyd_stop": ([_vp, _i32, _i32, _dbl, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_lloyd_train": ([_vp, _i32, _i64, _i32, _i32, _i32, _vp, _i32, _dbl, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_lloyd_final_objective": ([_vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_kmeanspp": ([_vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp], _i32),
    "cspq_crc32_workspace_bytes": ([_i64], ctypes.c_size_t),
    "cspq_crc32_device": ([_vp, _i64, ctypes.c_uint32, _vp, _vp, _vp], _i32),
    "cspq_crc32_combine": ([ctypes.c_uint32, ctypes.c_uint32, _i64], ctypes.c_uint32),
    "cspq_unpack_vecs": ([_vp, _i64, _i32, _i32, _i32, _i64, _vp, _vp, _vp], _i32),
    "cspq_adc_tables": ([_vp, _i64, _i32, _vp, _i32, _i32, _i32, _vp, _vp], _i32),
    "cspq_adc_scores": ([_vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp], _i32),
    "cspq_topn": ([_vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp], _i32),
    "cspq_exact_distances": ([_vp, _i64, _vp, _i64, _i32, _vp, _vp, _vp], _i32),
    "cspq_encode_vecs_file": ([ctypes.c_char_p, _i32, ctypes.c_char_p, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                               _i32, _i64, _i32, _i32, _vp, _vp], _i32),
}

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available: there is no
    CPU fallback for the product path."""


def build(force: bool = False) -> str:
    """Compile libcspq_b200.so for sm_100a with csrc/Makefile (nvcc)."""
    if force and os.path.exists(LIB_PATH):
        os.remove(LIB_PATH)
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], check=True)
    return LIB_PATH


def load():
    """Load (but do not build) the library; raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} not found: build it with __graft_entry__.build() "
                "(nvcc, sm_100a); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def header_symbols() -> list[str]:
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cspq_[a-z0-9_]+)\s*\(", txt)))


def call(name: str, *args):
    """Call an entry point and map its status to the package's exceptions."""
    rc = getattr(load(), name)(*args)
    if rc != CSPQ_OK:
        raise_status(rc, name)
    return rc


def raise_status(rc: int, name: str):
    """Raise the package exception for a non-zero CSPQ_E* status."""
    from .core import ConfigError, DataError, FormatError, TrainingError
    msg = load().cspq_last_error().decode(errors="replace")
    if rc == CSPQ_E_CONFIG:
        raise ConfigError(msg)
    if rc == CSPQ_E_DATA:
        raise DataError(msg)
    if rc == CSPQ_E_TRAINING:
        raise TrainingError(msg)
    if rc == CSPQ_E_FORMAT:
        raise FormatError(msg)
    raise RuntimeError(f"{name} failed ({rc}): {msg}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    load()
