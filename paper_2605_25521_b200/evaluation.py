"""Quality checks: reconstruction error and flat ADC recall against an exact
brute-force ground truth -- mirror of /root/reference/pkg/src/cspq/evaluation.py.

The heavy parts run on the GPU behind the C ABI (csrc/adc.cu): ADC lookup
tables, table-summed scores, exact lexsort-order top-N selection and the
float64 ground-truth distances.  Identical codes give identical reports
whatever kernel produced them, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._device import to_device
from .bulk import CodebookSet, ExecutionPlan, encode_dataset
from .core import ConfigError, CorruptionError, DataError, PQCodes
from .kernels import EncoderVariant

__all__ = ["EvalReport", "reconstruct", "reconstruct_all", "chunk_sqdist", "adc_tables", "adc_scores",
           "adc_search", "adc_search_batched", "exact_topn", "mse_of", "evaluate"]

_Q_CHUNK = 256  # queries per GPU pass (bounds the (queries, n) score / distance buffer)


@dataclass(frozen=True)
class EvalReport:
    mse: float
    recall_at_n: float
    top_n: int
    n_queries: int
    n_db: int
    variant: str

    def __post_init__(self):
        if not 0.0 <= self.recall_at_n <= 1.0:
            raise DataError(f"recall out of range: {self.recall_at_n}")
        if self.mse < 0.0:
            raise DataError(f"negative mse: {self.mse}")


def _torch():
    from ._device import torch
    return torch()


def _dev():
    from ._device import device
    N.require_cuda()
    return device(None)


def reconstruct(codes_row, codebooks) -> np.ndarray:
    """Inverse of encoding for one row: chunk j is centroid codes[j] (evaluation.py:37-49)."""
    cbset = CodebookSet.from_codebooks(codebooks)
    row = np.asarray(codes_row)
    if row.ndim != 1 or row.shape[0] != cbset.m:
        raise ConfigError(f"codes row shape {row.shape} does not match m={cbset.m}")
    if row.size and (int(row.max()) >= cbset.k or int(row.min()) < 0):
        raise CorruptionError(f"code out of range for k={cbset.k}")
    return np.ascontiguousarray(cbset.rowmajor[np.arange(cbset.m), row.astype(np.int64)].reshape(-1))


def _check_codes(codes: PQCodes, cbset: CodebookSet):
    if codes.m != cbset.m:
        raise ConfigError(f"codes m={codes.m} does not match codebooks m={cbset.m}")
    if codes.codes.size and int(codes.codes.max()) >= cbset.k:
        raise CorruptionError(f"code out of range for k={cbset.k}")


def _codes_array(codes: PQCodes, k: int) -> np.ndarray:
    """The codes in the width the scoring kernel reads for tables of k entries (uint8 for
    k <= 256); a code >= k would index past its table (IndexError in the reference)."""
    if codes.codes.size and int(codes.codes.max()) >= k:
        raise CorruptionError(f"code out of range for tables of k={k}")
    return np.ascontiguousarray(codes.codes, dtype=np.uint8 if k <= 256 else np.uint16)


def reconstruct_all(codes: PQCodes, codebooks) -> np.ndarray:
    """(n, d) reconstruction of every row (evaluation.py:52-62), gathered on the GPU."""
    cbset = CodebookSet.from_codebooks(codebooks)
    _check_codes(codes, cbset)
    t, dev = _torch(), _dev()
    return _reconstruct_dev(to_device(codes.codes, dev), cbset, dev).cpu().numpy()


def _reconstruct_dev(codes_t, cbset, dev):
    t = _torch()
    rm = to_device(cbset.rowmajor, dev)                              # (m, k, sub)
    j = t.arange(cbset.m, device=dev)[None, :]
    return rm[j, codes_t.long()].reshape(codes_t.shape[0], cbset.d)  # (n, m, sub) -> (n, d)


def chunk_sqdist(q_sub: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    """Float32 squared distances from one query chunk to (k, sub) centroids
    (evaluation.py:65-74, host helper, numpy's own arithmetic)."""
    diff = centroids - q_sub[None, :]
    return np.einsum("kt,kt->k", diff, diff)


def _tables_dev(Q, cbset, dev):
    t = _torch()
    from ._device import ptr, stream_ptr
    rm, _, _, _, _ = cbset.on_device(dev)
    T = t.empty((Q.shape[0], cbset.m, cbset.k), dtype=t.float32, device=dev)
    N.call("cspq_adc_tables", ptr(Q), Q.shape[0], cbset.d, ptr(rm), cbset.m, cbset.k, cbset.sub_dim, ptr(T),
           stream_ptr(dev))
    return T


def _queries(query, cbset, one: bool):
    q = np.ascontiguousarray(np.asarray(query, dtype=np.float32))
    if one:
        if q.ndim != 1 or q.shape[0] != cbset.d:
            raise ConfigError(f"query length {q.shape} does not match d={cbset.d}")
        return q[None, :]
    if q.ndim != 2 or q.shape[1] != cbset.d:
        raise ConfigError(f"queries shape {q.shape} does not match d={cbset.d}")
    return q


def adc_tables(query: np.ndarray, codebooks) -> np.ndarray:
    """Per-chunk lookup tables[j][l] = ||q_j - c_l||^2, float32 (evaluation.py:77-88)."""
    cbset = CodebookSet.from_codebooks(codebooks)
    q = _queries(query, cbset, True)
    t, dev = _torch(), _dev()
    return _tables_dev(to_device(q, dev), cbset, dev)[0].cpu().numpy()


def _scores_dev(T, codes_t, k, dev):
    t = _torch()
    from ._device import ptr, stream_ptr
    nq, m = T.shape[0], T.shape[1]
    S = t.empty((nq, codes_t.shape[0]), dtype=t.float32, device=dev)
    N.call("cspq_adc_scores", ptr(T), nq, ptr(codes_t), codes_t.shape[0], m, k, ptr(S), stream_ptr(dev))
    return S


def adc_scores(tables: np.ndarray, codes: PQCodes) -> np.ndarray:
    """Approximate squared distances, float32 table sums in chunk order (evaluation.py:91-96)."""
    t, dev = _torch(), _dev()
    T = to_device(np.asarray(tables, dtype=np.float32), dev)
    if T.dim() != 2 or T.shape[0] != codes.m:
        raise ConfigError(f"tables shape {tuple(T.shape)} does not match m={codes.m}")
    c = to_device(_codes_array(codes, T.shape[1]), dev)
    return _scores_dev(T[None], c, T.shape[1], dev)[0].cpu().numpy()


def _topn_dev(V, topn: int, dev):
    t = _torch()
    from ._device import ptr, stream_ptr
    nq, n = V.shape
    idx = t.empty((nq, topn), dtype=t.int64, device=dev)
    val = t.empty((nq, topn), dtype=V.dtype, device=dev)
    N.call("cspq_topn", ptr(V), V.element_size(), nq, n, topn, ptr(idx), ptr(val), stream_ptr(dev))
    return idx, val


def adc_search_batched(queries, codes: PQCodes, codebooks, topn: int):
    """Top-N database rows per query by table-summed asymmetric distance, in
    lexsort order (ties -> smaller index); topn clamped to the database size.
    Returns (indices (nq, topn) int64, distances (nq, topn) float32)."""
    cbset = CodebookSet.from_codebooks(codebooks)
    Q = _queries(queries, cbset, False)
    t, dev = _torch(), _dev()
    topn = min(int(topn), codes.n)
    if codes.n == 0 or topn <= 0:
        return np.empty((Q.shape[0], 0), np.int64), np.empty((Q.shape[0], 0), np.float32)
    c = to_device(_codes_array(codes, cbset.k), dev)
    Qd = to_device(Q, dev)
    I, D = [], []
    for lo in range(0, Q.shape[0], _Q_CHUNK):
        T = _tables_dev(Qd[lo:lo + _Q_CHUNK], cbset, dev)
        idx, val = _topn_dev(_scores_dev(T, c, cbset.k, dev), topn, dev)
        I.append(idx.cpu().numpy())
        D.append(val.cpu().numpy())
    return np.concatenate(I), np.concatenate(D)


def adc_search(query, codes: PQCodes, codebooks, topn: int):
    """One query (evaluation.py:106-117): (indices, approx_distances)."""
    cbset = CodebookSet.from_codebooks(codebooks)
    q = _queries(query, cbset, True)
    idx, d = adc_search_batched(q, codes, codebooks, topn)
    return idx[0], d[0]


def exact_topn(queries: np.ndarray, db: np.ndarray, topn: int) -> np.ndarray:
    """Ground-truth neighbour lists (evaluation.py:114-129): float32 inputs,
    float64 distances ||x||^2 - 2 q.x, ties broken by index -- on the GPU."""
    t, dev = _torch(), _dev()
    from ._device import ptr, stream_ptr
    Q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
    X = np.ascontiguousarray(np.asarray(db, dtype=np.float32))
    n = X.shape[0]
    topn = min(int(topn), n)
    if Q.shape[0] == 0 or topn <= 0:
        return np.empty((Q.shape[0], max(topn, 0)), np.int64)
    if Q.shape[1] != X.shape[1]:
        raise ConfigError(f"queries d={Q.shape[1]} does not match database d={X.shape[1]}")
    Xd = to_device(X, dev)
    nrm = t.empty(n, dtype=t.float64, device=dev)
    out = []
    for lo in range(0, Q.shape[0], _Q_CHUNK):
        Qd = to_device(Q[lo:lo + _Q_CHUNK], dev)
        Dd = t.empty((Qd.shape[0], n), dtype=t.float64, device=dev)
        N.call("cspq_exact_distances", ptr(Qd), Qd.shape[0], ptr(Xd), n, X.shape[1], ptr(nrm), ptr(Dd),
               stream_ptr(dev))
        out.append(_topn_dev(Dd, topn, dev)[0].cpu().numpy())
    return np.concatenate(out)


def mse_of(dataset, codes: PQCodes, codebooks) -> float:
    """Mean over vectors of ||v - reconstruct(encode(v))||^2 (evaluation.py:132-139):
    float32 difference, float64 squares and sums (order differs from numpy's:
    agreement to ~1e-15 relative)."""
    X = dataset.data if hasattr(dataset, "data") and not isinstance(dataset, np.ndarray) else np.asarray(
        dataset, dtype=np.float32)
    cbset = CodebookSet.from_codebooks(codebooks)
    _check_codes(codes, cbset)
    t, dev = _torch(), _dev()
    Xd = to_device(np.asarray(X, dtype=np.float32), dev)
    R = _reconstruct_dev(to_device(codes.codes, dev), cbset, dev)
    diff = (Xd - R).double()
    return float((diff * diff).sum(dim=1).sum().item() / max(X.shape[0], 1))


def evaluate(dataset, queries, codebooks, variant: EncoderVariant = EncoderVariant.BLOCKED, topn: int = 10, *,
             codes: PQCodes | None = None, groundtruth: np.ndarray | None = None, workers: int = 1) -> EvalReport:
    """Encode (or reuse codes), run flat ADC search, report MSE and recall (evaluation.py:142-180)."""
    X = dataset.data if hasattr(dataset, "data") and not isinstance(dataset, np.ndarray) else np.asarray(
        dataset, dtype=np.float32)
    Q = queries.data if hasattr(queries, "data") and not isinstance(queries, np.ndarray) else np.asarray(
        queries, dtype=np.float32)
    if Q.shape[0] == 0:
        raise DataError("empty query set")
    if codes is None:
        codes = encode_dataset(X, codebooks, ExecutionPlan(variant=variant, workers=workers))
    if groundtruth is None:
        groundtruth = exact_topn(Q, X, topn)
    gt = np.asarray(groundtruth)[:, :topn]
    idx, _ = adc_search_batched(Q, codes, codebooks, topn)
    hits = 0
    for a, b in zip(idx, gt):
        hits += len(set(a.tolist()) & set(int(v) for v in b))
    recall = hits / float(gt.shape[0] * gt.shape[1])
    return EvalReport(mse=mse_of(X, codes, codebooks), recall_at_n=recall, top_n=topn, n_queries=Q.shape[0],
                      n_db=X.shape[0], variant=variant.value)
