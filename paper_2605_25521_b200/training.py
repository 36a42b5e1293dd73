"""Per-subspace codebook training on the B200 -- the drop-in for
``cspq.training`` (/root/reference/pkg/src/cspq/training.py).

The reference trains subspaces one after another on the CPU (numpy/BLAS
float64 Lloyd, training.py:109-159, after k-means++ seeding,
training.py:76-92).  Here all M subspaces of a call are trained together
on the GPU: one batched k-means++ (``cspq_kmeanspp``) and one batched
Lloyd run (``cspq_lloyd_train``), each subspace keeping its own stop
decision, objective trace and iteration count.  Host-side work is limited
to what the reference also does with numpy's generator: the per-subspace
PCG64 streams (training.py:162-163), the row sample (training.py:166-172),
the seeding draws, and input validation.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._device import device, ptr, stream_ptr, to_device, torch
from .core import Codebook, DataError, TrainingError

__all__ = [
    "TrainConfig", "KMeansResult", "lloyd_iterate", "lloyd_iterate_batched", "run_lloyd",
    "kmeanspp_init_batched", "train_codebook", "train_codebook_report", "train_all_codebooks",
    "train_all_codebooks_report",
]


@dataclass(frozen=True)
class TrainConfig:
    """training.py:21-43: k, max_iters, tol (relative improvement stop), seed,
    sample_cap (None -> 256*k points per subspace; <= 0 -> all points)."""

    k: int = 256
    max_iters: int = 25
    tol: float = 1e-4
    seed: int = 0
    sample_cap: int | None = None

    def __post_init__(self):
        if self.k < 1:
            raise TrainingError(f"k must be >= 1, got {self.k}")
        if self.max_iters < 1:
            raise TrainingError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.tol < 0:
            raise TrainingError(f"tol must be >= 0, got {self.tol}")

    def resolved_cap(self) -> int | None:
        if self.sample_cap is None:
            return 256 * self.k
        return None if self.sample_cap <= 0 else self.sample_cap


@dataclass
class KMeansResult:
    """training.py:46-54: float32 centroids, objective trace (one value per
    iteration plus the final-pass objective), final assignments."""

    centroids: np.ndarray
    objectives: list[float] = field(default_factory=list)
    assignments: np.ndarray | None = None
    n_train: int = 0
    iterations: int = 0


def _stack_points(points_list):
    """[(n, sub)] -> (m, n, sub) contiguous, float32 when every value is
    exactly representable (the usual float64(float32) training input),
    else float64."""
    P = np.ascontiguousarray(np.stack([np.asarray(p, dtype=np.float64) for p in points_list]))
    P32 = P.astype(np.float32)
    if np.array_equal(P32.astype(np.float64), P, equal_nan=True):
        return P32, 0
    return P, 1


def lloyd_iterate_batched(points, init, cfg: TrainConfig, dev=None, *,
                          return_assignments: bool = True) -> list[KMeansResult]:
    """Lloyd from given float64 initial centroids for m subspaces at once.

    points: (m, n, sub) array (float32 or float64) or a list of (n, sub);
    init: (m, k, sub) float64.  Each subspace follows training.py:109-159
    exactly, including its own early stop.  ``return_assignments=False``
    leaves the final assignments on the device (KMeansResult.assignments is
    None): callers that only need the codebooks skip an (m, n) int64 copy."""
    N.require_cuda()
    t = torch()
    if isinstance(points, t.Tensor):  # device-resident (m, n, sub) float32/float64
        P = points.contiguous()
        pf64 = 1 if P.dtype == t.float64 else 0
        if P.dtype not in (t.float32, t.float64):
            P, pf64 = P.float(), 0
    elif isinstance(points, (list, tuple)) or np.asarray(points).dtype != np.float32:
        P, pf64 = _stack_points(points if isinstance(points, (list, tuple)) else list(np.asarray(points)))
    else:
        P, pf64 = np.ascontiguousarray(points, dtype=np.float32), 0
    C = np.array(init, dtype=np.float64, copy=True, order="C")
    m, n, sub = P.shape
    k = C.shape[1]
    if C.shape != (m, k, sub):
        raise TrainingError(f"initial centroids {C.shape} do not match points {P.shape}")
    dev = device() if dev is None else dev
    with t.cuda.device(dev):
        Pd = P if isinstance(P, t.Tensor) and P.device == dev else to_device(P, dev)
        Cd = to_device(C, dev)
        ws = t.zeros(N.load().cspq_lloyd_workspace_bytes(n, m, sub, k), dtype=t.uint8, device=dev)
        C32 = t.empty((m, k, sub), dtype=t.float32, device=dev)
        asg = t.empty((m, n), dtype=t.int32, device=dev)
        objs = t.zeros((m, cfg.max_iters + 1), dtype=t.float64, device=dev)
        iters = t.zeros((m,), dtype=t.int32, device=dev)
        N.call("cspq_lloyd_train", ptr(Pd), pf64, n, m, sub, k, ptr(Cd), cfg.max_iters, float(cfg.tol),
               ptr(C32), ptr(asg), ptr(objs), ptr(iters), ptr(ws), stream_ptr(dev))
        # assignments leave as one pinned int64 block (widened on the device); results slice it
        if return_assignments:
            asg64 = t.empty((m, n), dtype=t.int64, pin_memory=True)
            asg64.copy_(asg.long(), non_blocking=True)
        C32h, objh, ith = (x.cpu().numpy() for x in (C32, objs, iters))
        t.cuda.current_stream(dev).synchronize()
        asgh = asg64.numpy() if return_assignments else None
    out = []
    for j in range(m):
        it = int(ith[j])
        out.append(KMeansResult(centroids=np.ascontiguousarray(C32h[j]),
                                objectives=[float(v) for v in objh[j, :it + 1]],
                                assignments=None if asgh is None else asgh[j], n_train=n, iterations=it))
    return out


def lloyd_iterate(pts64: np.ndarray, centroids: np.ndarray, cfg: TrainConfig) -> KMeansResult:
    """training.py:109-159 for one subspace (float64 points, float64 init)."""
    P = np.asarray(pts64, dtype=np.float64)
    return lloyd_iterate_batched([P], np.asarray(centroids, dtype=np.float64)[None], cfg)[0]


def kmeanspp_init_batched(points_list, k: int, rngs, dev=None) -> np.ndarray:
    """training.py:76-92 for m subspaces: the host draws exactly what the
    reference draws from each generator (rng.integers(n), then one
    rng.random() per rng.choice), the GPU does the D^2 arithmetic.
    points_list: [(n, sub)] arrays, or an already stacked (m, n, sub) CUDA
    tensor (float32 or float64)."""
    N.require_cuda()
    t = torch()
    if isinstance(points_list, t.Tensor):
        P = points_list.contiguous()
        pf64 = 1 if P.dtype == t.float64 else 0
    else:
        P, pf64 = _stack_points(points_list)
    m, n, sub = P.shape
    states = [r.bit_generator.state for r in rngs]
    first = np.array([int(r.integers(n)) for r in rngs], dtype=np.int64)
    u = np.stack([r.random(k - 1) if k > 1 else np.zeros(0) for r in rngs]).astype(np.float64)
    u = np.ascontiguousarray(u.reshape(m, max(k - 1, 0)))
    dev = device() if dev is None else dev
    with t.cuda.device(dev):
        Pd = P if isinstance(P, t.Tensor) and P.device == dev else to_device(P, dev)
        fd = to_device(first, dev)
        ud = to_device(u if u.size else np.zeros((m, 1)), dev)
        C = t.zeros((m, k, sub), dtype=t.float64, device=dev)
        status = t.zeros((m,), dtype=t.int32, device=dev)
        ws = t.zeros(N.load().cspq_lloyd_workspace_bytes(n, m, sub, k), dtype=t.uint8, device=dev)
        N.call("cspq_kmeanspp", ptr(Pd), pf64, n, m, sub, k, ptr(fd), ptr(ud), ptr(C), ptr(status), ptr(ws),
               stream_ptr(dev))
        Ch, st = C.cpu().numpy(), status.cpu().numpy()
    if (st == 3).any():
        j = int(np.flatnonzero(st == 3)[0])
        raise DataError(f"subspace {j}: k-means++ D^2 mass is NaN (non-finite training points)")
    for j in np.flatnonzero(st < 0):
        # step c met zero D^2 mass (every remaining point coincides with a chosen centroid, e.g.
        # after float64 underflow): the reference draws rng.integers(n) for steps c..k-1
        # (training.py:84-86; d2 stays all-zero once it is).  Replay the generator exactly:
        # integers(n), c-1 random() draws, then the integer draws.
        c = int(-st[j])
        r = rngs[j]
        r.bit_generator.state = states[j]
        r.integers(n)
        if c > 1:
            r.random(c - 1)
        idx = [int(r.integers(n)) for _ in range(c, k)]
        src = P[j] if not isinstance(P, t.Tensor) else P[j].cpu().numpy()
        Ch[j, c:] = np.asarray(src, dtype=np.float64)[idx]
    return Ch


def _distinct_at_least(pts64: np.ndarray, k: int) -> bool:
    """np.unique(pts64, axis=0).shape[0] >= k (training.py:102-105) without sorting every
    row: rows go into a set until it holds k of them (a few hundred rows on real data).
    Adding 0.0 maps -0.0 to +0.0 so the bytes compare like np.unique's values do."""
    a = np.ascontiguousarray(pts64 + 0.0)
    rows = a.view(np.dtype((np.void, a.dtype.itemsize * a.shape[1]))).ravel()
    seen = set()
    for lo in range(0, rows.shape[0], 1024):
        seen.update(rows[lo:lo + 1024].tolist())
        if len(seen) >= k:
            return True
    return False


def _validate_points(pts64: np.ndarray, k: int):
    n = pts64.shape[0]
    if n < k:
        raise TrainingError(f"need at least k={k} training points, got {n}")
    if k > 1 and not _distinct_at_least(pts64, k):
        raise TrainingError(f"degenerate data: fewer than k={k} distinct training points")


def run_lloyd(points: np.ndarray, cfg: TrainConfig, rng: np.random.Generator) -> KMeansResult:
    """k-means++ seeding plus Lloyd for one subspace (training.py:95-106)."""
    pts64 = np.asarray(points, dtype=np.float64)
    _validate_points(pts64, cfg.k)
    init = kmeanspp_init_batched([pts64], cfg.k, [rng])
    return lloyd_iterate_batched([pts64], init, cfg)[0]


def _subspace_rngs(seed: int, m: int) -> list[np.random.Generator]:
    """training.py:162-163: one PCG64 stream per subspace."""
    return [np.random.Generator(np.random.PCG64(s)) for s in np.random.SeedSequence(seed).spawn(m)]


def _sample(points: np.ndarray, cap: int | None, rng: np.random.Generator) -> np.ndarray:
    """training.py:166-172: sorted sample without replacement when above the cap."""
    if cap is None or points.shape[0] <= cap:
        return points
    idx = rng.choice(points.shape[0], size=cap, replace=False)
    idx.sort()
    return points[idx]


def _train_many(subspace_points, cfg: TrainConfig, rngs, labels, return_assignments: bool = True):
    """Sample, validate, seed and train a list of subspaces together."""
    # every subspace has its own generator, so the draws and gathers run on host threads
    # (numpy releases the GIL in both) with exactly the reference's per-stream draw order
    cap = cfg.resolved_cap()
    jobs = list(zip(subspace_points, rngs))
    if len(jobs) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(min(len(jobs), os.cpu_count() or 1)) as ex:
            samples = list(ex.map(lambda pr: _sample(pr[0], cap, pr[1]), jobs))
    else:
        samples = [_sample(p, cap, r) for p, r in jobs]
    P = None
    if all(s.dtype == np.float32 for s in samples) and len({s.shape for s in samples}) == 1:
        # float32 data (every configuration): float64(x) is exact and injective there, so the
        # count / distinct checks give the reference's answers on the float32 rows and the stack
        # needs no float64 round trip (~0.7 s of host time for c3-shaped data)
        P32 = np.ascontiguousarray(np.stack(samples))
        if np.isfinite(P32).all():
            for s, j in zip(P32, labels):
                try:
                    _validate_points(s, cfg.k)
                except (TrainingError, DataError) as exc:
                    raise type(exc)(f"subspace {j}: {exc}") from None
            P = P32
    if P is None:
        sampled = []
        for s, j in zip(samples, labels):
            try:
                s64 = np.asarray(s, dtype=np.float64)
                _validate_points(s64, cfg.k)
            except (TrainingError, DataError) as exc:
                raise type(exc)(f"subspace {j}: {exc}") from None
            sampled.append(s64)
        P, _ = _stack_points(sampled)
    # move to the GPU once; both stages read the tensor
    dev = device()
    Pd = to_device(P, dev)
    init = kmeanspp_init_batched(Pd, cfg.k, rngs, dev)
    return lloyd_iterate_batched(Pd, init, cfg, dev, return_assignments=return_assignments)


def train_codebook(subvectors: np.ndarray, cfg: TrainConfig, subspace_index: int = 0) -> Codebook:
    return train_codebook_report(subvectors, cfg, subspace_index)[0]


def train_codebook_report(subvectors: np.ndarray, cfg: TrainConfig,
                          subspace_index: int = 0) -> tuple[Codebook, KMeansResult]:
    """training.py:180-194: the subspace's own generator is the
    (subspace_index)-th child of SeedSequence(cfg.seed)."""
    pts = np.asarray(subvectors, dtype=np.float32)
    if pts.ndim != 2:
        raise TrainingError(f"training points must be 2-D, got shape {pts.shape}")
    if not np.isfinite(pts).all():
        raise DataError(f"non-finite training data in subspace {subspace_index}")
    rng = _subspace_rngs(cfg.seed, subspace_index + 1)[subspace_index]
    s = _sample(pts, cfg.resolved_cap(), rng)
    s64 = np.asarray(s, dtype=np.float64)
    _validate_points(s64, cfg.k)
    init = kmeanspp_init_batched([s64], cfg.k, [rng])
    res = lloyd_iterate_batched([s64], init, cfg)[0]
    return Codebook.from_rowmajor(subspace_index, res.centroids), res


def train_all_codebooks(dataset, params, cfg: TrainConfig) -> list[Codebook]:
    # (the reports' assignments are not returned: they stay on the device)
    return _train_all(dataset, params, cfg, return_assignments=False)[0]


def train_all_codebooks_report(dataset, params, cfg: TrainConfig):
    return _train_all(dataset, params, cfg, return_assignments=True)


def _train_all(dataset, params, cfg: TrainConfig, return_assignments: bool):
    """training.py:203-224: one codebook per subspace from its own sample.
    Accepts a VectorDataset or a raw (n, d) array (the reference's
    ``hasattr(dataset, "data")`` probe mistakes an ndarray's buffer for a
    dataset -- SURVEY §0.6; here raw arrays simply work)."""
    data = dataset.data if isinstance(getattr(dataset, "data", None), np.ndarray) else np.asarray(dataset, dtype=np.float32)
    if data.shape[1] != params.d:
        raise TrainingError(f"dataset dimensionality {data.shape[1]} does not match d={params.d}")
    rngs = _subspace_rngs(cfg.seed, params.m)
    sub = params.sub_dim
    # column views: _sample gathers only the sampled rows (the same arrays the reference's
    # per-subspace slice + sample produce, without copying every column block first)
    pts = [data[:, j * sub:(j + 1) * sub] for j in range(params.m)]
    reports = _train_many(pts, cfg, rngs, range(params.m), return_assignments)
    return [Codebook.from_rowmajor(j, r.centroids) for j, r in enumerate(reports)], reports
