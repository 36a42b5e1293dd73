"""CPU oracle wrapper -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker or the timed CPU baseline.  The product package
(``paper_2605_25521_b200``) never imports it.

The arithmetic lives in ``oracle/pq_oracle.c`` (strict IEEE fp32 encode,
float64 Lloyd), a restatement of the reference's ``cspq`` kernels
(/root/reference/pkg/src/cspq/kernels.py:84-316, training.py:57-159).  It is
pinned against golden vectors generated from the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz; checked by
tests/test_oracle_golden.py).

Also here: the near-tie classifier of the reference's ``run_verify``
(cli.py:194-201) and ``mse_of`` (evaluation.py:134-139), restated in numpy.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpq_oracle.so")
_lib = None

VARIANT_REFERENCE = 0
VARIANT_REFORM = 1
VARIANT_NOBIAS = 2


def build() -> str:
    """Compile the oracle with oracle/Makefile (gcc, strict IEEE)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "pq_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.oracle_encode.argtypes = [vp, i32, i64, i32, vp, vp, i32, i32, i32, i32, vp, i32, vp, i32]
        L.oracle_encode.restype = i32
        L.oracle_lloyd.argtypes = [vp, i64, i32, vp, i32, i32, ctypes.c_double, vp, vp, vp, vp, i32]
        L.oracle_lloyd.restype = i32
        L.oracle_pairwise_sum.argtypes = [vp, i64]
        L.oracle_pairwise_sum.restype = ctypes.c_double
        L.oracle_einsum_dot.argtypes = [vp, vp, i32]
        L.oracle_einsum_dot.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def encode(X, rowmajor, biases, variant: int = VARIANT_REFORM, want_best: bool = False,
           threads: int = 0):
    """codes (n, m) of X (n, d) f32 or u8 against codebooks (m, k, sub)."""
    X = np.ascontiguousarray(X)
    in_u8 = 1 if X.dtype == np.uint8 else 0
    if not in_u8:
        X = np.ascontiguousarray(X, dtype=np.float32)
    CB = np.ascontiguousarray(rowmajor, dtype=np.float32)
    B = np.ascontiguousarray(biases, dtype=np.float32)
    m, k, sub = CB.shape
    n = X.shape[0]
    dtype = np.uint8 if k <= 256 else np.uint16
    codes = np.empty((n, m), dtype=dtype)
    best = np.empty((n, m), dtype=np.float32) if want_best else None
    rc = lib().oracle_encode(
        _ptr(X), in_u8, n, X.shape[1], _ptr(CB), _ptr(B), m, k, sub, variant, _ptr(codes),
        codes.itemsize, _ptr(best) if want_best else None, int(threads),
    )
    if rc != 0:
        raise ValueError(f"oracle_encode rc={rc}")
    return (codes, best) if want_best else codes


def lloyd(pts64, init64, max_iters: int, tol: float, threads: int = 0):
    """training.py:109-159 for one subspace.  Returns a dict with centroids
    (f32), centroids64, objectives, assignments (int64), iterations."""
    P = np.ascontiguousarray(pts64, dtype=np.float64)
    C = np.array(init64, dtype=np.float64, copy=True, order="C")
    n, sub = P.shape
    k = C.shape[0]
    objs = np.empty(max_iters + 1, dtype=np.float64)
    assign = np.empty(n, dtype=np.int64)
    cast = np.empty((k, sub), dtype=np.float32)
    iters = ctypes.c_int(0)
    nobj = lib().oracle_lloyd(
        _ptr(P), n, sub, _ptr(C), k, int(max_iters), float(tol), _ptr(objs), _ptr(assign),
        _ptr(cast), ctypes.byref(iters), int(threads),
    )
    if nobj < 0:
        raise ValueError(f"oracle_lloyd rc={nobj}")
    return {
        "centroids": cast,
        "centroids64": C,
        "objectives": objs[:nobj].tolist(),
        "assignments": assign,
        "iterations": iters.value,
    }


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().oracle_pairwise_sum(_ptr(a), a.shape[0]))


def einsum_dot(a, b) -> float:
    """np.einsum("t,t->") order for one float64 row pair (oracle_einsum_dot)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return float(lib().oracle_einsum_dot(_ptr(a), _ptr(b), a.shape[0]))


def compute_biases(rowmajor) -> np.ndarray:
    """core.py:232-243: 0.5*||c||^2 accumulated in float64, stored float32."""
    a = np.asarray(rowmajor, dtype=np.float32)
    return (0.5 * np.einsum("...kt,...kt->...k", a, a, dtype=np.float64)).astype(np.float32)


def classify_mismatches(X, rowmajor, codes_a, codes_b, tolerance: float = 1e-5):
    """The reference's verify rule (cli.py:194-201): a disagreement at (i, j)
    is a near-tie when the float64 distances of the two codes differ by at
    most tolerance * max(1, larger distance); anything else is a failure.
    Returns (n_mismatch, n_near_tie, n_failure, worst_rel_gap)."""
    X = np.asarray(X)
    CB = np.asarray(rowmajor, dtype=np.float64)
    m, k, sub = CB.shape
    ii, jj = np.nonzero(np.asarray(codes_a) != np.asarray(codes_b))
    near = fail = 0
    worst = 0.0
    for i, j in zip(ii.tolist(), jj.tolist()):
        v = X[i, j * sub:(j + 1) * sub].astype(np.float64)
        da = float(((CB[j, int(codes_a[i, j])] - v) ** 2).sum())
        db = float(((CB[j, int(codes_b[i, j])] - v) ** 2).sum())
        gap = abs(da - db)
        rel = gap / max(1.0, da, db)
        worst = max(worst, rel)
        if gap <= tolerance * max(1.0, da, db):
            near += 1
        else:
            fail += 1
    return len(ii), near, fail, worst


def mse_of(X, codes, rowmajor) -> float:
    """evaluation.py:134-139: mean over rows of ||x - reconstruct(code)||^2."""
    X = np.asarray(X)
    CB = np.asarray(rowmajor, dtype=np.float32)
    m, k, sub = CB.shape
    recon = np.concatenate([CB[j][np.asarray(codes)[:, j].astype(np.int64)] for j in range(m)], axis=1)
    diff = (X.astype(np.float32) - recon).astype(np.float64)
    return float(np.einsum("it,it->i", diff, diff).sum() / max(X.shape[0], 1))
