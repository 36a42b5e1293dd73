"""Verification and ablation-bench harness of the encode path.

Mirrors the two harness functions of the reference's ``cspq.cli`` that drive
the hot path (the CLI's argument parsing, plots and file plumbing stay out of
scope):

* ``run_verify`` (cli.py:174-229): three-way encoder equivalence
  (REFERENCE / REFORMULATED / BLOCKED) over sampled vectors; every
  disagreement is classified with the same float64 rule -- a near-tie when
  the reference top-2 gap is within ``tolerance * max(1, second_best)``, a
  failure otherwise.
* ``run_bench_matrix`` (cli.py:232-276): the four-stage ablation (formula,
  order, bias precomputation) timed through ``encode_dataset``, median of
  ``reps`` after one warm-up, speed-ups against the first row.
  ``BenchResult`` / ``BENCH_CSV_COLUMNS`` / ``write_bench_csv`` follow
  cli.py:45-72, 279-284.

Every encode runs on the GPU through the C ABI (``encode_dataset``); here the
order / w / workers knobs only label the rows (codes are plan-invariant) and
the variant and bias precomputation select the kernel (REFERENCE -> the
generic exact kernel, BLOCKED without precomputed biases -> the recomputed
bias tables)."""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass

import numpy as np

from .bulk import CHUNK_MAJOR, VECTOR_MAJOR, CodebookSet, ExecutionPlan, encode_dataset
from .kernels import EncoderVariant, native_lane_width

__all__ = ["BENCH_CSV_COLUMNS", "BenchResult", "run_bench_matrix", "run_verify", "write_bench_csv"]

BENCH_CSV_COLUMNS = [
    "variant", "order", "w", "block_size",
    "n", "d", "m", "k", "wall_seconds", "vps", "speedup",
]


@dataclass
class BenchResult:
    """One row of the ablation matrix (cli.py:51-72)."""

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

    def csv_row(self) -> list:
        return [
            self.variant, self.order, self.w, self.block_size,
            self.n, self.d, self.m, self.k,
            f"{self.wall_seconds:.6f}",
            f"{self.vectors_per_second:.1f}",
            f"{self.speedup_vs_baseline:.4f}",
        ]


def _rows_of(dataset) -> np.ndarray:
    # the reference probes hasattr(dataset, "data"), which on an ndarray picks
    # its raw buffer; accept arrays and VectorDatasets alike
    X = dataset.data if isinstance(getattr(dataset, "data", None), np.ndarray) else dataset
    X = np.asarray(X)
    return X if X.dtype == np.uint8 else np.asarray(X, dtype=np.float32)


def run_bench_matrix(dataset, codebooks, w: int | None = None, block_size: int = 4096,
                     workers: int = 1, reps: int = 3) -> list[BenchResult]:
    """The four-stage ablation (cli.py:232-276): baseline order/formula
    through the full pipeline; rows 3 and 4 differ only in bias
    precomputation.  Wall time of ``encode_dataset`` on host rows (H2D, GPU
    encode, D2H), median of ``reps`` after one warm-up."""
    cbset = CodebookSet.from_codebooks(codebooks)
    X = _rows_of(dataset)
    wv = w if w is not None else native_lane_width()
    rows = [
        ("reference", VECTOR_MAJOR, EncoderVariant.REFERENCE, True),
        ("blocked", VECTOR_MAJOR, EncoderVariant.BLOCKED, False),
        ("blocked", CHUNK_MAJOR, EncoderVariant.BLOCKED, False),
        ("blocked+reform", CHUNK_MAJOR, EncoderVariant.BLOCKED, True),
    ]
    results = []
    baseline = None
    for label, order, variant, precomp in rows:
        plan = ExecutionPlan(order=order, block_size=block_size, variant=variant, w=wv, workers=workers)
        encode_dataset(X, cbset, plan, precomputed_bias=precomp)  # warm-up
        times = []
        for _ in range(max(1, reps)):
            t0 = time.perf_counter()
            encode_dataset(X, cbset, plan, precomputed_bias=precomp)
            times.append(time.perf_counter() - t0)
        wall = float(np.median(times))
        if baseline is None:
            baseline = wall
        results.append(BenchResult(
            variant=label, order=order, w=wv, block_size=block_size,
            n=X.shape[0], d=X.shape[1], m=cbset.m, k=cbset.k,
            wall_seconds=wall, vectors_per_second=X.shape[0] / wall,
            speedup_vs_baseline=baseline / wall,
        ))
    return results


def write_bench_csv(results, path) -> None:
    """cli.py:279-284."""
    with open(path, "w", newline="") as f:
        writer = csv.writer(f)
        writer.writerow(BENCH_CSV_COLUMNS)
        for r in results:
            writer.writerow(r.csv_row())


def run_verify(dataset, codebooks, samples: int, tolerance: float, seed: int = 0,
               w: int | None = None, workers: int = 1):
    """Three-way encoder equivalence over sampled vectors (cli.py:174-229).

    Returns ``(checked, near_ties, failures, details)``; ``details`` lists
    ``(vector, chunk, kind, gap, codes)`` per disagreement, ``codes`` mapping
    each variant's name to its code."""
    X = _rows_of(dataset)
    cbset = CodebookSet.from_codebooks(codebooks)
    rng = np.random.Generator(np.random.PCG64(seed))
    if samples < X.shape[0]:
        idx = rng.choice(X.shape[0], size=samples, replace=False)
        idx.sort()
        X = np.ascontiguousarray(X[idx])
    outs = {}
    for variant in EncoderVariant:
        plan = ExecutionPlan(variant=variant, w=w, workers=workers)
        outs[variant] = encode_dataset(X, cbset, plan).codes
    ref = outs[EncoderVariant.REFERENCE]
    disagree = np.zeros(ref.shape, dtype=bool)
    for variant in (EncoderVariant.REFORMULATED, EncoderVariant.BLOCKED):
        disagree |= outs[variant] != ref
    near_ties = 0
    failures = 0
    details = []
    sub = cbset.sub_dim
    for i, j in zip(*np.nonzero(disagree)):
        v = X[i, j * sub:(j + 1) * sub].astype(np.float64)
        cents = cbset.rowmajor[j].astype(np.float64)
        dists = np.einsum("kt,kt->k", cents - v[None, :], cents - v[None, :])
        top2 = np.partition(dists, 1)[:2]
        gap = float(top2[1] - top2[0])
        if gap <= tolerance * max(1.0, float(top2[1])):
            near_ties += 1
            kind = "near-tie"
        else:
            failures += 1
            kind = "failure"
        details.append((int(i), int(j), kind, gap, {v_.name: int(outs[v_][i, j]) for v_ in EncoderVariant}))
    return X.shape[0], near_ties, failures, details
