"""Multi-GPU sharding of the hot path: one process per GPU,
``torch.distributed`` (NCCL on B200, gloo in the CPU tests) for the plumbing.

* Encode shards rows with no data-path collective: every rank encodes its
  contiguous row range with the codebooks rank 0 broadcast once
  (``broadcast_codebooks``).  Codes are identical for any world size because
  rows are independent (the reference's plan invariance, test_bulk.py:44-62).
* Lloyd (training.py:109-159) has one exchange step per iteration.  Every
  rank holds the (small) training sample; rank r assigns its row shard, then
  either
    - ``reduce="allgather"`` (default): the assignment and objective terms of
      all shards are all-gathered and every rank runs the point-ordered
      accumulation, update, repair and stop rule on identical data -- the
      result is bit-identical to the single-GPU run (and to the oracle) for
      every world size; or
    - ``reduce="allreduce"`` (the north_star's scheme): each rank accumulates
      its shard's point-ordered sums / counts / pairwise objective and one
      all-reduce(sum) combines them; the mean is then identical up to float64
      summation order (not bit-identical across world sizes).  If any cluster
      is empty the assignments are gathered for the exact teleport.

The per-iteration compute goes through a backend object so the collective
logic is testable on CPU: ``CudaSteps`` calls the C ABI
(include/cspq_b200.h); tests plug in a numpy backend.
"""

from __future__ import annotations

import numpy as np

from .training import KMeansResult, TrainConfig

__all__ = ["shard_range", "broadcast_codebooks", "encode_sharded", "lloyd_sharded", "CudaSteps"]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row range [begin, end) of ``rank``."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    return dist


def broadcast_codebooks(rowmajor, src: int = 0, group=None):
    """Broadcast a (m, k, sub) float32 codebook tensor from ``src`` (in place)."""
    dist = _dist()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(rowmajor, src=src, group=group)
    return rowmajor


def encode_sharded(X_local, codebooks, plan=None, group=None):
    """Encode this rank's rows (a CUDA tensor) with the broadcast codebooks;
    no collective on the data path.  Returns the local codes tensor."""
    from .bulk import encode_dataset_device
    return encode_dataset_device(X_local, codebooks, plan)


class CudaSteps:
    """Lloyd step backend on the CUDA library (batched over subspaces)."""

    def __init__(self, P, pf64: int, n: int, m: int, sub: int, k: int, dev):
        from . import _native as N
        from ._device import torch
        t = torch()
        self.N, self.t = N, t
        self.P, self.pf64, self.n, self.m, self.sub, self.k, self.dev = P, pf64, n, m, sub, k, dev
        self.ws = t.zeros(N.load().cspq_lloyd_workspace_bytes(n, m, sub, k), dtype=t.uint8, device=dev)

    def _sp(self):
        from ._device import stream_ptr
        return stream_ptr(self.dev)

    def empty(self, shape, kind):
        t = self.t
        dt = {"f64": t.float64, "i32": t.int32}[kind]
        return t.zeros(shape, dtype=dt, device=self.dev)

    def assign(self, C64, state, b, e, assign, sq):
        p = lambda x: x.data_ptr()
        self.N.call("cspq_lloyd_assign", p(self.P), self.pf64, self.n, self.m, self.sub, self.k, p(C64),
                    p(state), b, e, p(assign), p(sq), p(self.ws), self._sp())

    def accumulate(self, state, assign, sq, b, e, counts, sums, obj):
        p = lambda x: x.data_ptr()
        self.N.call("cspq_lloyd_accumulate", p(self.P), self.pf64, self.n, self.m, self.sub, self.k, p(state),
                    p(assign), p(sq), b, e, p(counts), p(sums), p(obj), p(self.ws), self._sp())

    def update(self, counts, sums, state, C64, empties, nempty):
        p = lambda x: x.data_ptr()
        self.N.call("cspq_lloyd_update", p(counts), p(sums), self.m, self.k, self.sub, p(state), p(C64),
                    p(empties), p(nempty), self._sp())

    def repair(self, assign, state, empties, nempty, C64):
        p = lambda x: x.data_ptr()
        self.N.call("cspq_lloyd_repair", p(self.P), self.pf64, self.n, self.m, self.sub, self.k, p(assign),
                    p(state), p(empties), p(nempty), p(C64), p(self.ws), self._sp())

    def stop(self, obj, max_iters, tol, state, prev, iterations, objectives):
        p = lambda x: x.data_ptr()
        self.N.call("cspq_lloyd_stop", p(obj), self.m, max_iters, float(tol), p(state), p(prev),
                    p(iterations), p(objectives), self._sp())

    def finish(self, C64, max_iters, iterations, objectives):
        """float32 cast, REFERENCE final pass and final objective (training.py:143-154)."""
        t, N = self.t, self.N
        p = lambda x: x.data_ptr()
        C32 = C64.float()
        P32 = self.P.float() if self.pf64 else self.P
        asg = t.empty((self.m, self.n), dtype=t.int32, device=self.dev)
        N.call("cspq_encode_subspace_major", p(P32), self.n, self.m, self.sub, p(C32), p(C32), self.k, p(asg),
               N.VARIANT_REFERENCE, self._sp())
        fobj = t.empty((self.m,), dtype=t.float64, device=self.dev)
        N.call("cspq_lloyd_final_objective", p(self.P), self.pf64, self.n, self.m, self.sub, self.k, p(C32),
               p(asg), p(fobj), p(self.ws), self._sp())
        objectives[t.arange(self.m, device=self.dev), iterations.long()] = fobj
        return C32, asg


def _all_gather_rows(x, n: int, world: int, group):
    """Concatenate every rank's row shard [b_r, e_r) of x (..., n) along the last axis."""
    dist = _dist()
    import torch
    chunks = [shard_range(n, r, world) for r in range(world)]
    width = max(e - b for b, e in chunks)
    rank = dist.get_rank(group)
    b, e = chunks[rank]
    send = torch.zeros(x.shape[:-1] + (width,), dtype=x.dtype, device=x.device)
    send[..., :e - b] = x[..., b:e]
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    for r, (rb, re_) in enumerate(chunks):
        x[..., rb:re_] = recv[r][..., :re_ - rb]
    return x


def lloyd_sharded(steps, init64, cfg: TrainConfig, group=None, reduce: str = "allgather") -> list[KMeansResult]:
    """Row-sharded Lloyd for m subspaces (see module doc).  ``steps`` is a
    CudaSteps (or a test backend) over the full (m, n, sub) sample; init64 is
    (m, k, sub) float64 on the backend's device."""
    dist = _dist()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m, n, k, sub = steps.m, steps.n, steps.k, steps.sub
    b, e = shard_range(n, rank, world)
    C64 = init64.clone()
    state = steps.empty((m,), "i32") + 1
    prev = steps.empty((m,), "f64") + float("inf")
    iterations = steps.empty((m,), "i32")
    objectives = steps.empty((m, cfg.max_iters + 1), "f64")
    assign = steps.empty((m, n), "i32")
    sq = steps.empty((m, n), "f64")
    counts = steps.empty((m, k), "f64")
    sums = steps.empty((m, k, sub), "f64")
    obj = steps.empty((m,), "f64")
    empties = steps.empty((m, k), "i32")
    nempty = steps.empty((m,), "i32")
    for _ in range(cfg.max_iters):
        steps.assign(C64, state, b, e, assign, sq)
        if reduce == "allgather":
            if world > 1:
                _all_gather_rows(assign, n, world, group)
                _all_gather_rows(sq, n, world, group)
            steps.accumulate(state, assign, sq, 0, n, counts, sums, obj)
        else:
            steps.accumulate(state, assign, sq, b, e, counts, sums, obj)
            if world > 1:  # one fused all-reduce of (counts, sums, objective partials)
                import torch
                buf = torch.cat([counts.flatten(), sums.flatten(), obj.flatten()])
                dist.all_reduce(buf, group=group)
                counts.copy_(buf[:m * k].view(m, k))
                sums.copy_(buf[m * k:m * k + m * k * sub].view(m, k, sub))
                obj.copy_(buf[m * k + m * k * sub:].view(m))
        steps.update(counts, sums, state, C64, empties, nempty)
        if reduce != "allgather" and world > 1 and bool((nempty > 0).any()):
            _all_gather_rows(assign, n, world, group)  # exact teleport needs every residual
        steps.repair(assign, state, empties, nempty, C64)
        steps.stop(obj, cfg.max_iters, cfg.tol, state, prev, iterations, objectives)
        if not bool((state > 0).any()):
            break
    C32, final_asg = steps.finish(C64, cfg.max_iters, iterations, objectives)
    C32h = C32.cpu().numpy()
    asgh = final_asg.cpu().numpy()
    objh = objectives.cpu().numpy()
    ith = iterations.cpu().numpy()
    return [KMeansResult(centroids=np.ascontiguousarray(C32h[j]),
                         objectives=[float(v) for v in objh[j, :int(ith[j]) + 1]],
                         assignments=asgh[j].astype(np.int64), n_train=n, iterations=int(ith[j]))
            for j in range(m)]
