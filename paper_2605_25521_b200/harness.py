"""Encoder-equivalence check and ablation timing on the GPU path.

The reference drives its hot path from two harness functions in
``cspq.cli`` (its acceptance criterion 5 runs them): ``run_verify``
(cli.py:174-229) and ``run_bench_matrix`` (cli.py:232-276), with
``BenchResult`` / ``write_bench_csv`` (cli.py:45-72, 279-284) as their
output format.  Their return values and CSV layout are the contract kept
here; the work is organised for the GPU:

* verify: the sample is uploaded once, the three encoder variants run on the
  device (``encode_dataset_device``), the disagreement mask is formed there,
  and only the disagreeing (vector, subspace) pairs come back.  Their float64
  top-2 gaps are computed in one vectorised pass that reproduces
  ``np.einsum("kt,kt->k")``'s summation order (``einsum_rowsq``), so gaps and
  the near-tie / failure split equal the reference's bit for bit
  (tests/golden/verify_golden.npz).
* bench matrix: the ablation is a table of ``Stage`` rows (formula, order,
  bias precomputation); each is timed end to end through the public
  ``encode_dataset`` on host rows (H2D, encode, D2H), median of ``reps``
  after one warm-up.  On the GPU the order / w / workers knobs only label a
  row -- codes are plan-invariant -- while variant and bias precomputation
  select the kernel.
"""

from __future__ import annotations

import csv
import time
from dataclasses import astuple, dataclass, fields

import numpy as np

from ._device import device, torch
from .bulk import CHUNK_MAJOR, VECTOR_MAJOR, CodebookSet, ExecutionPlan, encode_dataset, encode_dataset_device
from .kernels import EncoderVariant, native_lane_width

__all__ = ["BENCH_CSV_COLUMNS", "BenchResult", "run_bench_matrix", "run_verify", "write_bench_csv", "einsum_rowsq"]


@dataclass
class BenchResult:
    """One ablation row; field order = CSV column order (cli.py:51-72)."""

    variant: str
    order: str
    w: int
    block_size: int
    n: int
    d: int
    m: int
    k: int
    wall_seconds: float
    vectors_per_second: float
    speedup_vs_baseline: float

    # printf formats of the three measured columns; the rest print as-is
    _FMT = {"wall_seconds": "{:.6f}", "vectors_per_second": "{:.1f}", "speedup_vs_baseline": "{:.4f}"}

    def csv_row(self) -> list:
        return [self._FMT[f.name].format(v) if f.name in self._FMT else v
                for f, v in zip(fields(self), astuple(self))]


# the CSV header names the two ratio columns by their short names
BENCH_CSV_COLUMNS = [f.name for f in fields(BenchResult)][:9] + ["vps", "speedup"]


@dataclass(frozen=True)
class Stage:
    """One row of the ablation: which formula, traversal order and bias handling."""

    label: str
    order: str
    variant: EncoderVariant
    precomputed_bias: bool


# cli.py:240-246: baseline formula in vector-major order, then the blocked formula, then
# chunk-major order, then precomputed biases (rows 3 and 4 differ only in the bias)
ABLATION = (
    Stage("reference", VECTOR_MAJOR, EncoderVariant.REFERENCE, True),
    Stage("blocked", VECTOR_MAJOR, EncoderVariant.BLOCKED, False),
    Stage("blocked", CHUNK_MAJOR, EncoderVariant.BLOCKED, False),
    Stage("blocked+reform", CHUNK_MAJOR, EncoderVariant.BLOCKED, True),
)


def _host_rows(dataset) -> np.ndarray:
    """float32 (or uint8) host rows of a VectorDataset or an array."""
    X = dataset.data if isinstance(getattr(dataset, "data", None), np.ndarray) else dataset
    X = np.asarray(X)
    return X if X.dtype == np.uint8 else np.asarray(X, dtype=np.float32)


def _median_wall(fn, reps: int) -> float:
    fn()  # warm-up (codebook upload, pipeline buffers)
    walls = []
    for _ in range(max(1, reps)):
        t0 = time.perf_counter()
        fn()
        walls.append(time.perf_counter() - t0)
    return float(np.median(walls))


def run_bench_matrix(dataset, codebooks, w: int | None = None, block_size: int = 4096,
                     workers: int = 1, reps: int = 3) -> list[BenchResult]:
    """Time every ``ABLATION`` stage through ``encode_dataset`` on host rows;
    speed-ups are against the first stage."""
    cbset = CodebookSet.from_codebooks(codebooks)
    X = _host_rows(dataset)
    n, d = X.shape
    lane_w = native_lane_width() if w is None else w
    walls = []
    for st in ABLATION:
        plan = ExecutionPlan(order=st.order, block_size=block_size, variant=st.variant, w=lane_w, workers=workers)
        walls.append(_median_wall(lambda: encode_dataset(X, cbset, plan, precomputed_bias=st.precomputed_bias), reps))
    return [BenchResult(st.label, st.order, lane_w, block_size, n, d, cbset.m, cbset.k, wall, n / wall, walls[0] / wall)
            for st, wall in zip(ABLATION, walls)]


def write_bench_csv(results, path) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerows([BENCH_CSV_COLUMNS] + [r.csv_row() for r in results])


def einsum_rowsq(diff: np.ndarray) -> np.ndarray:
    """sum_t diff[..., t]**2 in float64 with np.einsum's own order (numpy's 2-lane
    sum_of_products: 8-element blocks folded back to front into two lane accumulators, a
    tail of lane pairs, then lane0 + lane1 -- oracle_einsum_dot in oracle/pq_oracle.c),
    vectorised over the leading axes."""
    p = diff * diff
    s = p.shape[-1]
    lanes = [np.zeros(p.shape[:-1]), np.zeros(p.shape[:-1])]
    t = 0
    while s - t >= 8:
        for lane in (0, 1):
            for q in (6, 4, 2, 0):
                lanes[lane] = p[..., t + q + lane] + lanes[lane]
        t += 8
    while t < s:
        lanes[0] = p[..., t] + lanes[0]
        if t + 1 < s:
            lanes[1] = p[..., t + 1] + lanes[1]
        t += 2
    return lanes[0] + lanes[1]


def run_verify(dataset, codebooks, samples: int, tolerance: float, seed: int = 0,
               w: int | None = None, workers: int = 1):
    """Encoder equivalence on ``samples`` sampled vectors (PCG64(seed), sorted).
    Returns ``(checked, near_ties, failures, details)`` with one
    ``(vector, subspace, "near-tie" | "failure", gap, {variant name: code})`` per
    disagreement of REFORMULATED or BLOCKED with REFERENCE, in row-major order; a
    disagreement is a near-tie when the float64 top-2 distance gap is at most
    ``tolerance * max(1, second best)``."""
    t = torch()
    X = _host_rows(dataset)
    cbset = CodebookSet.from_codebooks(codebooks)
    if samples < X.shape[0]:
        pick = np.random.Generator(np.random.PCG64(seed)).choice(X.shape[0], size=samples, replace=False)
        X = np.ascontiguousarray(X[np.sort(pick)])
    dev = device()
    Xd = t.from_numpy(X if X.flags.writeable else X.copy()).to(dev)
    codes = {v: encode_dataset_device(Xd, cbset, ExecutionPlan(variant=v, w=w, workers=workers))
             for v in EncoderVariant}
    base = codes[EncoderVariant.REFERENCE]
    mask = (codes[EncoderVariant.REFORMULATED] != base) | (codes[EncoderVariant.BLOCKED] != base)
    ij = t.nonzero(mask).cpu().numpy()  # row-major, like np.nonzero
    if ij.shape[0] == 0:
        return X.shape[0], 0, 0, []
    got = {v: c[mask].cpu().numpy().view(np.uint16 if cbset.k > 256 else np.uint8) for v, c in codes.items()}
    rows, subs = ij[:, 0], ij[:, 1]
    s = cbset.sub_dim
    V = X.reshape(X.shape[0], cbset.m, s)[rows, subs].astype(np.float64)           # (q, s)
    C = cbset.rowmajor[subs].astype(np.float64)                                     # (q, k, s)
    D = einsum_rowsq(C - V[:, None, :])                                             # (q, k)
    top2 = np.sort(D, axis=1)[:, :2] if D.shape[1] > 1 else np.repeat(D, 2, axis=1)
    gaps = top2[:, 1] - top2[:, 0]
    near = gaps <= tolerance * np.maximum(1.0, top2[:, 1])
    details = [(int(i), int(j), "near-tie" if nt else "failure", float(g),
                {v.name: int(got[v][q]) for v in EncoderVariant})
               for q, (i, j, nt, g) in enumerate(zip(rows, subs, near, gaps))]
    return X.shape[0], int(near.sum()), int((~near).sum()), details
