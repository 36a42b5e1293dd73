"""Multi-process (world size 2, gloo on CPU) tests of the sharded Lloyd
driver and the encode sharding helpers.  The per-step compute uses a numpy
backend with the CUDA kernels' semantics (test-only), so the collective
logic -- shard ranges, all-gather of assignments, fused all-reduce of the
statistics, exact empty-cluster teleport -- runs without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_25521_b200.distributed import broadcast_codebooks, lloyd_sharded, shard_range
from paper_2605_25521_b200.training import TrainConfig


class NumpySteps:
    """CPU stand-in for distributed.CudaSteps (same arguments, same semantics)."""

    def __init__(self, P64, k):
        self.P = P64  # (m, n, sub) float64 numpy
        self.m, self.n, self.sub = P64.shape
        self.k = k

    def empty(self, shape, kind):
        return torch.zeros(shape, dtype=torch.float64 if kind == "f64" else torch.int32)

    def assign(self, C64, state, b, e, assign, sq):
        C = C64.numpy()
        for j in range(self.m):
            if not state[j]:
                continue
            x = self.P[j, b:e]
            cn = np.einsum("kt,kt->k", C[j], C[j])
            d = cn[None, :] - 2.0 * (x @ C[j].T)
            a = np.argmin(d, axis=1)
            assign[j, b:e] = torch.from_numpy(a.astype(np.int32))
            v = d[np.arange(e - b), a] + np.einsum("it,it->i", x, x)
            sq[j, b:e] = torch.from_numpy(np.maximum(v, 0.0))

    def accumulate(self, state, assign, sq, b, e, counts, sums, obj):
        for j in range(self.m):
            if not state[j]:
                continue
            a = assign[j, b:e].numpy().astype(np.int64)
            cnt = np.bincount(a, minlength=self.k).astype(np.float64)
            s = np.zeros((self.k, self.sub))
            np.add.at(s, a, self.P[j, b:e])
            counts[j] = torch.from_numpy(cnt)
            sums[j] = torch.from_numpy(s)
            obj[j] = float(sq[j, b:e].numpy().sum())

    def update(self, counts, sums, state, C64, empties, nempty):
        for j in range(self.m):
            if not state[j]:
                continue
            c = counts[j].numpy()
            ne = c > 0
            C64[j][torch.from_numpy(ne)] = torch.from_numpy(sums[j].numpy()[ne] / c[ne, None])
            em = np.flatnonzero(~ne)
            nempty[j] = len(em)
            empties[j, :len(em)] = torch.from_numpy(em.astype(np.int32))

    def repair(self, assign, state, empties, nempty, C64):
        for j in range(self.m):
            if not state[j] or int(nempty[j]) == 0:
                continue
            a = assign[j].numpy().astype(np.int64)
            C = C64[j].numpy()
            diff = self.P[j] - C[a]
            r = np.einsum("it,it->i", diff, diff)
            for q in range(int(nempty[j])):
                cand = int(np.argmax(r))
                C64[j, int(empties[j, q])] = torch.from_numpy(self.P[j, cand].copy())
                r[cand] = -1.0

    def stop(self, obj, max_iters, tol, state, prev, iterations, objectives):
        for j in range(self.m):
            if not state[j]:
                continue
            o = float(obj[j])
            objectives[j, int(iterations[j])] = o
            iterations[j] += 1
            p = float(prev[j])
            stop = o == 0.0 or (p < np.inf and (p - o) <= tol * max(p, 1e-300))
            prev[j] = o
            if stop or int(iterations[j]) >= max_iters:
                state[j] = 0

    def finish(self, C64, max_iters, iterations, objectives):
        C32 = C64.float()
        asg = torch.zeros((self.m, self.n), dtype=torch.int32)
        for j in range(self.m):
            c = C32[j].numpy().astype(np.float64)
            d = ((self.P[j][:, None, :] - c[None, :, :]) ** 2).sum(-1)
            a = np.argmin(d, axis=1)
            asg[j] = torch.from_numpy(a.astype(np.int32))
            diff = self.P[j] - c[a]
            objectives[j, int(iterations[j])] = float(np.einsum("it,it->i", diff, diff).sum())
        return C32, asg


def _data(seed=3):
    rng = np.random.default_rng(seed)
    m, n, sub, k = 3, 701, 4, 16
    cen = rng.uniform(-4, 4, size=(m, k, sub))
    P = np.stack([cen[j][rng.integers(0, k, n)] + rng.normal(0, 0.5, (n, sub)) for j in range(m)])
    P = P.astype(np.float32).astype(np.float64)
    init = P[:, :k].copy()
    init[:, 3] = init[:, 2]  # duplicate init -> an empty cluster in the first iteration
    return P, init, k


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P, init, k = _data()
        res = lloyd_sharded(NumpySteps(P, k), torch.from_numpy(init), TrainConfig(k=k, max_iters=15, tol=1e-6),
                            reduce=mode)
        cb = torch.arange(12, dtype=torch.float32).reshape(1, 3, 4) * (1 if rank == 0 else 0)
        broadcast_codebooks(cb)
        out[rank] = ([r.centroids.tobytes() for r in res], [r.objectives for r in res],
                     [r.iterations for r in res], cb.numpy().tobytes())
    finally:
        dist.destroy_process_group()


def _run(world, mode):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, mode, out), nprocs=world, join=True)
        return dict(out)


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def test_allgather_mode_is_world_size_invariant():
    one = _run(1, "allgather")[0]
    two = _run(2, "allgather")
    for rank in (0, 1):
        assert two[rank][0] == one[0]   # centroids bit-identical
        assert two[rank][1] == one[1]   # objective traces identical
        assert two[rank][2] == one[2]
        assert two[rank][3] == two[0][3]  # codebooks broadcast from rank 0


def test_allreduce_mode_matches_to_summation_order():
    one = _run(1, "allreduce")[0]
    two = _run(2, "allreduce")
    assert two[0][0] == two[1][0]  # every rank ends with the same centroids
    for a, b in zip(one[0], two[0][0]):
        ca, cb = np.frombuffer(a, np.float32), np.frombuffer(b, np.float32)
        assert np.allclose(ca, cb, rtol=1e-6, atol=1e-6)
    assert one[2] == two[0][2]
    for oa, ob in zip(one[1], two[0][1]):
        np.testing.assert_allclose(oa, ob, rtol=1e-12)
