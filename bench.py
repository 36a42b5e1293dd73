#!/usr/bin/env python
"""bench.py -- PQ-encoded vectors/s on B200 (BASELINE.json metric).

Headline workload (default): BASELINE config 3 -- N = 10,000,000
unit-normalised float32 rows, D = 768, M = 96 subspaces (d_sub = 8), K = 256,
codebooks from 10 Lloyd iterations (GPU, fp64) on a 200,000-row seeded sample.
A "step" is one encode pass of the rank's rows (one fused kernel launch).
Scaling is STRONG for c2-c5: the config's N rows are sharded across the ranks
(distributed.shard_range), so at 8 GPUs each encodes 1,250,000 of c3's 10M rows.
c1 (0.1 ms of work) runs replicas (weak).  With N > 1 the codebooks are
trained row-sharded with one all-gather per Lloyd iteration, bit-identical to
the single-GPU training (--reduce allreduce: the north_star's one-all-reduce
scheme, equal up to float64 summation order); encode has no data-path collective.

At N = 1 the same JSON line also carries ``extra``: the other BASELINE configs
measured in the same run -- c2 (train + encode per step), c4 (200M u8 rows,
device-resident and end to end), c5 (streaming 4,096-row batches from pinned
host memory, p50/p99 batch latency) -- each with its own parity spot check,
clock record and CPU baseline.

Launch: python bench.py [--gpus N --steps K --warmup W]
        torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)
        python bench.py --impl reference ...   (the reference's CPU encoder, host cores)

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PQ-encoded vectors/sec"
FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.45: SMs x FP32 lanes x FMA x max clock
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--rows", type=int, default=0, help="total rows (0 = the config's N); per rank with weak scaling")
    p.add_argument("--scaling", choices=["auto", "weak", "strong"], default="auto",
                   help="auto: strong (the config's N sharded across ranks) for c2-c5, weak replicas for c1")
    p.add_argument("--mode", default="auto", choices=["auto", "exact", "guarded"])
    p.add_argument("--e2e-rows", type=int, default=0,
                   help="rows per rank through the host API (0 = max(2M, 6 GB of rows), or the whole shard for c5)")
    p.add_argument("--streams", type=int, default=0, help="host pipeline streams (0 = 3, or 2 for c5: 4096-row batches saturate PCIe with two in flight; more only queue -- p50 0.87 ms at 2, 1.81 ms at 6, same vec/s)")
    p.add_argument("--e2e-batch", type=int, default=0,
                   help="host pipeline batch rows (0 = max(131072 rows, 256 MB) capped at a quarter of the sample, "
                        "or 4096 for c5)")
    p.add_argument("--train", choices=["auto", "sharded", "rank0"], default="auto",
                   help="codebook training: auto = fused cspq_lloyd_train at N = 1, row-sharded at N > 1; "
                        "rank0 = fused training on rank 0 + broadcast")
    p.add_argument("--reduce", choices=["allgather", "allreduce"], default="allgather",
                   help="sharded Lloyd exchange: allgather (bit-exact for any N, default) or allreduce (north_star "
                        "scheme: one all-reduce of counts/sums/objective, equal up to float64 summation order)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the c2/c4/c5 records at N = 1")
    p.add_argument("--extra-configs", default="c2,c4,c5")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--ref-seconds", type=float, default=150.0,
                   help="--impl reference: CPU budget of the whole warmup + steps run")
    return p.parse_args(argv)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def scaling_of(args, cfg):
    if args.scaling != "auto":
        return args.scaling
    return "weak" if cfg.name == "c1" else "strong"


def rows_of(args, cfg, ws, rank):
    """(begin, end, global rows) of this rank."""
    from paper_2605_25521_b200.distributed import shard_range
    total = args.rows or cfg.n
    if scaling_of(args, cfg) == "strong":
        b, e = shard_range(total, rank, ws)
        return b, e, total
    return rank * total, (rank + 1) * total, total * ws


def workload_desc(cfg, rows_local, global_rows, ws, scaling):
    per = (f"{rows_local:,} rows/GPU, global {global_rows:,}" if scaling == "strong"
           else f"{rows_local:,} rows/GPU (replicas), global {global_rows:,}")
    return (f"{cfg.name}: {'u8' if cfg.dtype == 'u8' else 'f32'} rows D={cfg.d}, M={cfg.m} (d_sub={cfg.sub}), "
            f"K={cfg.k}, {per} ({scaling} scaling, {ws} GPU{'s' if ws > 1 else ''}), codebooks: "
            + (f"{cfg.iters} Lloyd iters on a {cfg.n_train:,}-row sample" if cfg.codebook == "lloyd"
               else "256 distinct data subvectors per subspace")
            + ("; a step = codebook training (all subspaces) + encode of all rows" if cfg.name == "c2" else ""))


def peaks():
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(mp))
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6547.2, 1590.0, "B200_PROFILING.md fallback"


# ----------------------------------------------------------------------------------- CPU baselines
def reference_module():
    """The unmodified reference package installed into baseline/_ref (pip --target), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "cspq")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cspq_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import cspq  # noqa: F401
        from cspq import bulk, core, training
        return {"bulk": bulk, "core": core, "training": training}
    except Exception:
        return None


def ref_encoder(rm, bs):
    """-> (encode(X) -> codes, description) with the reference's own encode_dataset, or the port."""
    cores = os.cpu_count() or 1
    R = reference_module()
    if R is not None:
        cset = R["bulk"].CodebookSet.from_codebooks([R["core"].Codebook.from_rowmajor(j, rm[j]) for j in range(rm.shape[0])])
        plan = R["bulk"].ExecutionPlan(workers=cores)
        return (lambda X: R["bulk"].encode_dataset(X, cset, plan).codes), "reference", \
            f"cspq.bulk.encode_dataset(X, codebooks, ExecutionPlan(workers={cores})) -- the unmodified reference " \
            f"(numba nogil threads) from baseline/_ref"
    from oracle import oracle as O
    return (lambda X: O.encode(X, rm, bs, O.VARIANT_REFORM, threads=cores)), "port", \
        f"oracle/pq_oracle.c strict-fp32 restatement of the reference encoder, OpenMP over {cores} threads"


def port_encoder(rm, bs):
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    return lambda X: O.encode(X, rm, bs, O.VARIANT_REFORM, threads=cores)


def time_cpu(enc, gen, seconds, cap_rows, min_rows=4096):
    """Rows/s of ``enc`` on a bounded prefix sized for ~``seconds`` of CPU work (re-sized
    until a run takes at least half the budget or covers ``cap_rows``)."""
    warm = gen(min(min_rows, cap_rows))
    enc(warm)  # JIT / thread-pool warm-up
    t0 = time.perf_counter()
    enc(warm)
    per_row = (time.perf_counter() - t0) / warm.shape[0]
    for _ in range(4):
        rows = int(max(min_rows, min(cap_rows, seconds / max(per_row, 1e-9))))
        X = gen(rows)
        t0 = time.perf_counter()
        enc(X)
        dt = time.perf_counter() - t0
        per_row = dt / rows
        if dt >= 0.5 * seconds or rows >= cap_rows:
            break
    return rows / dt, rows, dt


def cpu_baseline_record(cfg, rm, bs, gen, seconds):
    cores = os.cpu_count() or 1
    enc, kind, what = ref_encoder(rm, bs)
    cap = cfg.n if cfg.name in ("c1", "c2", "c5") else min(cfg.n, 1_000_000)  # 1M prefix c3/c4
    rate, rows, dt = time_cpu(enc, gen, seconds, cap)
    rec = {"value": rate, "unit": "vectors/s", "cores": cores, "kind": kind,
           "sample": f"{rows:,}-row prefix of {cfg.name} in {dt:.1f} s: {what}"}
    if kind == "reference":
        prate, prows, pdt = time_cpu(port_encoder(rm, bs), gen, seconds / 2, cap)
        rec["port"] = {"value": prate, "unit": "vectors/s", "cores": cores,
                       "sample": f"{prows:,} rows in {pdt:.1f} s (oracle/pq_oracle.c, OpenMP)"}
    return rec


def cpu_train_record(cfg, Ssm, init):
    """Reference training on one subspace (lloyd_iterate, numpy + OpenBLAS), x M subspaces."""
    import numpy as np
    p0 = Ssm[0].double().cpu().numpy()
    R = reference_module()
    t0 = time.perf_counter()
    if R is not None:
        tr = R["training"]
        tr.lloyd_iterate(p0, init[0].copy(), tr.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0))
        kind, what = "reference", "cspq.training.lloyd_iterate (numpy/OpenBLAS)"
    else:
        from oracle import oracle as O
        O.lloyd(p0, init[0], cfg.iters, 0.0)
        kind, what = "port", "oracle.lloyd (C, OpenMP)"
    one = time.perf_counter() - t0
    return {"seconds": one * cfg.m, "kind": kind, "cores": os.cpu_count() or 1,
            "sample": f"{what} on subspace 0 ({cfg.n_train:,} x {cfg.sub} fp64, {cfg.iters} iters, tol 0) "
                      f"in {one:.2f} s, x {cfg.m} subspaces (the reference trains them sequentially)"}


# ----------------------------------------------------------------------------------- reference arm
def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU encoder (cspq.bulk.encode_dataset from
    baseline/_ref, numba threads = all host cores; the C port if it is absent) on rank 0,
    same config / metric, a bounded prefix per step."""
    if rank != 0:
        return
    import numpy as np
    import torch

    from paper_2605_25521_b200 import configs as C
    cfg = C.CONFIGS[args.config]
    cuda = torch.cuda.is_available()
    dev = torch.device("cuda", 0) if cuda else torch.device("cpu")
    cores = os.cpu_count() or 1
    # codebooks: the config's own (trained) ones -- on the GPU, the training is bit-identical to the
    # reference's lloyd_iterate (tests/test_lloyd_full_gpu.py); it is setup, not the timed path
    note = "trained codebooks (GPU Lloyd, bit-identical to cspq.training.lloyd_iterate)"
    if cfg.codebook == "sampled":
        rm = C.sampled_codebooks(cfg, C.generate(cfg, 0, cfg.n, dev).cpu().numpy())
        note = "sampled codebooks (c1)"
    elif cuda:
        import paper_2605_25521_b200 as P
        Ssm = C.subspace_major(C.training_sample(cfg, dev), cfg.m)
        res = P.lloyd_iterate_batched(Ssm, C.lloyd_init(cfg, Ssm), P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0))
        rm = np.stack([r.centroids for r in res])
        del Ssm
    else:  # CPU-only contract check: the Lloyd initial points
        rm = C.lloyd_init(cfg, C.subspace_major(C.training_sample(cfg, dev), cfg.m)).astype(np.float32)
        note = "Lloyd initial points (no GPU to train on)"
    rm = np.ascontiguousarray(rm, dtype=np.float32)
    from oracle.oracle import compute_biases
    bs = compute_biases(rm)
    enc, kind, what = ref_encoder(rm, bs)
    cap = cfg.n if cfg.name in ("c1", "c2", "c5") else min(cfg.n, 1_000_000)
    gen = lambda r: C.generate(cfg, 0, r, dev).cpu().numpy()
    # size each step so that warmup + steps fit the budget
    rate0, _, _ = time_cpu(enc, gen, 2.0, cap)
    rows = int(max(4096, min(cap, args.ref_seconds / max(1, args.steps + args.warmup) * rate0)))
    X = gen(rows)
    for _ in range(args.warmup):
        enc(X)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        enc(X)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = rows / (ms / 1e3)
    scope = "encode"
    train = None
    if cfg.name == "c2":  # the config's scope is train + encode
        S = C.training_sample(cfg, dev)
        Ssm = C.subspace_major(S, cfg.m)
        init = C.lloyd_init(cfg, Ssm)
        train = cpu_train_record(cfg, Ssm, init)
        value = cfg.n / (train["seconds"] + cfg.n / value)
        scope = "train + encode (training: one subspace timed x M; encode: rows/s of the sampled steps x N)"
    sample = f"{rows:,}-row prefix of {cfg.name} per step: {what}"
    line = {
        "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling_of(args, cfg),
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_desc(cfg, cfg.n, cfg.n, 1, scaling_of(args, cfg)), "rows_per_step": rows,
                   "codebooks": note, "scope": scope},
        "cpu_baseline": {"value": value, "unit": "vectors/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if train is not None:
        line["train"] = train
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------- B200 arm
def count_launches(fn):
    """This library's kernel launches in one call of ``fn`` (cspq_launch_count: a host-side
    counter bumped at every launch site of libcspq_b200.so)."""
    from paper_2605_25521_b200 import _native as N
    L = N.load()
    L.cspq_launch_count(1)
    fn()
    return int(L.cspq_launch_count(1))


def train_codebooks(cfg, args, ws, rank, dev, timed_train=False):
    """-> (rowmajor (m, k, sub) float32 CUDA tensor identical on every rank, info dict)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_25521_b200 as P
    from paper_2605_25521_b200 import configs as C
    rm = torch.empty((cfg.m, cfg.k, cfg.sub), dtype=torch.float32, device=dev)
    info = {"train_s": None}
    sharded = args.train == "sharded" or (args.train == "auto" and ws > 1)
    if cfg.codebook == "sampled":
        if rank == 0:
            rm.copy_(torch.from_numpy(C.sampled_codebooks(cfg, C.generate(cfg, 0, cfg.n, dev).cpu().numpy())))
        info["mode"] = "sampled codebooks" + (" on rank 0 + broadcast" if ws > 1 else "")
    elif sharded:
        from paper_2605_25521_b200.distributed import CudaSteps, lloyd_sharded
        Ssm = C.subspace_major(C.training_sample(cfg, dev), cfg.m).contiguous()
        init = torch.from_numpy(C.lloyd_init(cfg, Ssm)).to(dev)
        steps = CudaSteps(Ssm, 0, cfg.n_train, cfg.m, cfg.sub, cfg.k, dev)
        tcfg = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
        lloyd_sharded(steps, init, P.TrainConfig(k=cfg.k, max_iters=1, tol=0.0), reduce=args.reduce)  # warm-up
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = lloyd_sharded(steps, init, tcfg, reduce=args.reduce)
        info["train_s"] = time.perf_counter() - t0
        rm.copy_(torch.from_numpy(np.stack([r.centroids for r in res])))
        info["mode"] = (f"row-sharded x{ws}, one {'all-gather (bit-exact)' if args.reduce == 'allgather' else 'all-reduce'}"
                        f" per iteration" if ws > 1 else "row-sharded driver at world size 1 (no collective)")
        info["results"] = res
        del Ssm
    else:
        if rank == 0:
            Ssm = C.subspace_major(C.training_sample(cfg, dev), cfg.m)
            init = C.lloyd_init(cfg, Ssm)
            P.lloyd_iterate_batched(Ssm, init, P.TrainConfig(k=cfg.k, max_iters=1, tol=0.0))  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = P.lloyd_iterate_batched(Ssm, init, P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0))
            info["train_s"] = time.perf_counter() - t0
            rm.copy_(torch.from_numpy(np.stack([r.centroids for r in res])))
            info["results"] = res
            del Ssm
        info["mode"] = "fused cspq_lloyd_train" + (" on rank 0 + NCCL broadcast" if ws > 1 else "")
    if ws > 1:
        dist.broadcast(rm, src=0)
    return rm, info


def codebook_set(rm):
    import paper_2605_25521_b200 as P
    rmh = rm.cpu().numpy()
    return P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rmh[j]) for j in range(rmh.shape[0])])


def encode_parity(cfg, X, out, cs, rows, dev, nrows=20_000):
    import numpy as np
    import torch

    from oracle import oracle as O
    rng = np.random.default_rng(123)
    idx = np.sort(rng.choice(rows, min(rows, nrows), replace=False))
    ti = torch.from_numpy(idx).to(dev)
    want = O.encode(X[ti].cpu().numpy(), cs.rowmajor, cs.biases, O.VARIANT_REFORM)
    got = out[ti].cpu().numpy()
    return {"rows_checked": int(idx.shape[0]), "code_mismatches": int((got != want).sum()),
            "against": "oracle/pq_oracle.c (pinned bit-exact to the reference's codes, tests/test_oracle_golden.py)"}


def train_parity(cfg, dev, results, subspaces=(0, 1)):
    """The GPU-trained centroids of a few subspaces against the oracle's Lloyd."""
    import numpy as np

    from oracle import oracle as O
    from paper_2605_25521_b200 import configs as C
    Ssm = C.subspace_major(C.training_sample(cfg, dev), cfg.m)
    init = C.lloyd_init(cfg, Ssm)
    worst, exact = 0.0, True
    for j in subspaces:
        o = O.lloyd(Ssm[j].double().cpu().numpy(), init[j], cfg.iters, 0.0)
        r = results[j]
        a, b = r.centroids.astype(np.float64), o["centroids"].astype(np.float64)
        rel = float((np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-30)).max())
        worst = max(worst, rel)
        exact = exact and r.centroids.tobytes() == o["centroids"].tobytes() and r.objectives == o["objectives"]
    return {"subspaces_checked": list(subspaces), "max_centroid_rel_err": worst, "bitexact": bool(exact),
            "against": "oracle Lloyd (pinned bit-exact to the reference's lloyd_iterate at full size, "
                       "tests/test_lloyd_full_gpu.py)"}


def timed_device_steps(step, steps, warmup, ws, dev, local, flush=None):
    """Warm-up, then ``steps`` calls bracketed by barrier + synchronize; CUDA events on the
    launching stream; NVML clocks sampled during the region.  -> (total_ms max over ranks,
    per-step ms, clocks)."""
    import torch
    import torch.distributed as dist

    from paper_2605_25521_b200.telemetry import ClockSampler
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        step()
    clocks = ClockSampler(local, period=0.01).start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for s in range(steps):
        if flush is not None:
            flush.fill_(s & 0xff)
        ev[2 * s].record(stream)
        step()
        ev[2 * s + 1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [ev[2 * s].elapsed_time(ev[2 * s + 1]) for s in range(steps)]
    total_ms = sum(step_ms) if flush is not None else ev[0].elapsed_time(ev[-1])
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), step_ms, clk


def e2e_record(cfg, args, X, cs, out, ws, dev, steps, train_fn=None, train_h2d=0):
    """Public host API with pinned buffers: H2D of the step's rows, encode, D2H of the codes,
    per step (c5: the whole shard in 4,096-row batches).  train_fn (c2): the training from the
    host-resident (pinned) sample runs inside every step and returns the codebooks the step
    encodes with; train_h2d = its host->device bytes."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_25521_b200 as P
    rows = X.shape[0]
    row_bytes = cfg.d * cfg.elem_bytes
    ne = min(args.e2e_rows or (rows if cfg.batch else max(2_000_000, (6 << 30) // row_bytes)), rows)
    batch_rows = cfg.batch or args.e2e_batch or max(1 << 17, (256 << 20) // row_bytes)
    if not (cfg.batch or args.e2e_batch):
        batch_rows = min(batch_rows, max(1 << 14, -(-ne // 4)))
    Xh = P.pinned_empty((ne, cfg.d), np.uint8 if cfg.dtype == "u8" else np.float32)
    Xh[:] = X[:ne].cpu().numpy()
    codes_h = P.pinned_empty((ne, cfg.m), np.uint8)
    eplan = P.ExecutionPlan(mode=args.mode, batch_rows=batch_rows, streams=args.streams or (2 if cfg.batch else 3))
    nb = (ne + batch_rows - 1) // batch_rows
    bms = np.zeros(nb, np.float64)
    P.encode_dataset_host(Xh, cs, eplan, out=codes_h)  # warm the pipeline
    if train_fn is not None:
        cs = train_fn()
    from paper_2605_25521_b200.telemetry import ClockSampler
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    lat = []
    clocks = ClockSampler(dev.index, period=0.01).start()
    t0 = time.perf_counter()
    for _ in range(steps):
        if train_fn is not None:
            cs = train_fn()
        P.encode_dataset_host(Xh, cs, eplan, out=codes_h, batch_ms=bms)
        lat.append(bms.copy())
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    clk = clocks.stop()
    if ws > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    e2e_val = ne * ws * steps / float(el.item())
    assert np.array_equal(codes_h[:4096], out[:4096].cpu().numpy()), "e2e codes differ from device codes"
    lat = np.concatenate(lat)
    rec = {"value": e2e_val, "unit": "vectors/s", "h2d_bytes_per_step": (int(ne * row_bytes) + train_h2d) * ws,
           "d2h_bytes_per_step": int(ne * cfg.m) * ws, "rows_per_gpu": ne, "batch_rows": batch_rows,
           "streams": eplan.streams,
           "batch_latency_ms": {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                                "batches": int(lat.shape[0]),
                                "def": f"device events: H2D start -> D2H end of one batch ({eplan.streams} batches in flight)"},
           "h2d_GBps": ne * row_bytes * steps / float(el.item()) / 1e9,
           "path": "encode_dataset_host (pinned numpy -> cspq_encode_host: multi-stream H2D/encode/D2H pipeline)",
           "clocks": clk, "steps": steps, "timing": "host wall clock around the steps, max over ranks"}
    if train_fn is not None:
        rec["path"] = "lloyd_iterate_batched (pinned host sample, KMeansResult back to host) + " + rec["path"]
    del Xh, codes_h
    return rec


def roofline_record(cfg, args, rows, ms_per_step, dev):
    import torch
    hbm, bf16, psrc = peaks()
    flops_launch = rows * cfg.flops_per_vec()
    achieved = flops_launch / (ms_per_step / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "encode_traffic.json")
    tc = args.mode in ("auto", "tensor") and cfg.k == 256 and cfg.sub in (4, 8)
    try:
        tj = json.load(open(tp))
        bpr = tj.get(cfg.name + ("_tc" if tc else ""), {}).get("dram_bytes_per_row")
        traffic = None if bpr is None else int(bpr * rows)
    except Exception:
        traffic = None
    f16_peak = bf16  # kind::f16 MMAs with fp32 accumulation run at the bf16 rate
    k_eff = 32 if cfg.sub == 8 else 16
    rec = {"bound": "fp32", "achieved": achieved, "peak": FP32_NOMINAL_TFLOPS, "unit": "TFLOP/s",
           "frac": achieved / FP32_NOMINAL_TFLOPS, "traffic": traffic,
           "kernel": ("encode_tc_kernel (tcgen05 kind::f16 on fp16 hi/lo splits + exact epilogue)" if tc else
                      "encode_k256_kernel (" + ("exact" if args.mode == "exact" else "guarded FFMA") + ")"),
           "peak_source": "north_star roofline = the slower of FP32 FFMA and tensor peaks: nominal FP32 "
                          "148 SMs x 128 lanes x 2 flop x 1.965 GHz (no FP32 entry in MEASURED_PEAKS.json)",
           "algorithmic_flops_per_row": cfg.flops_per_vec(), "algorithmic_bytes_per_row": cfg.bytes_per_vec(),
           "hbm_frac": (rows * cfg.bytes_per_vec() / (ms_per_step / 1e3) / 1e9) / hbm,
           "hbm_peak_gbs": hbm, "hbm_peak_source": psrc}
    if tc:
        rec["tensor"] = {
            "peak_f16_tflops": f16_peak, "peak_source": f"{psrc} bf16_tflops",
            "algorithmic_frac": achieved / f16_peak,
            "executed_tensor_tflops": achieved * (k_eff / cfg.sub),
            "executed_frac": achieved * (k_eff / cfg.sub) / f16_peak,
            "note": f"the MMA executes K={k_eff} fp16 per (row, subspace) for {cfg.sub} useful MACs "
                    "(hi/lo split + folded bias); the kernel is bound by issue slots: a half-rate ALU-pipe "
                    "instruction (the epilogue's FMNMX3) holds a sub-partition's issue port for two cycles"}
        alu_peak = torch.cuda.get_device_properties(dev).multi_processor_count * 4 * 16 * 1.965e9
        alu_ops = rows * cfg.m * cfg.k / (ms_per_step / 1e3)
        rec["alu"] = {"algorithmic_min_lane_ops_per_row": cfg.m * cfg.k, "achieved_lane_ops_per_s": alu_ops,
                      "peak_lane_ops_per_s": alu_peak, "frac": alu_ops / alu_peak,
                      "note": "FMNMX3 lane-ops of the two exact min trees only (K per (row, subspace)); "
                              "ncu's ALU-pipe busy fraction covers the rest (profiles/)"}
    return rec


def run_config(cfg, args, ws, rank, local, dev, steps, warmup, cpu_seconds, headline):
    """Measure one config; returns the record (rank 0) or None."""
    import numpy as np
    import torch

    import paper_2605_25521_b200 as P
    from paper_2605_25521_b200 import _native as N
    from paper_2605_25521_b200 import configs as C
    scaling = scaling_of(args, cfg)
    b, e, global_rows = rows_of(args, cfg, ws, rank)
    rows = e - b
    X = C.generate(cfg, b, e, dev)
    rm, tinfo = train_codebooks(cfg, args, ws, rank, dev)
    cs = codebook_set(rm)
    plan = P.ExecutionPlan(mode=args.mode)
    out = P.encode_dataset_device(X, cs, plan)
    torch.cuda.synchronize()
    parity = encode_parity(cfg, X, out, cs, rows, dev) if rank == 0 else None

    train_step = None
    if cfg.name == "c2":  # the config's timed scope: codebook training + encode of all rows
        from paper_2605_25521_b200.distributed import CudaSteps, lloyd_sharded
        Ssm = C.subspace_major(C.training_sample(cfg, dev), cfg.m).contiguous()
        init_np = C.lloyd_init(cfg, Ssm)
        tcfg = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
        if ws > 1:
            init_d = torch.from_numpy(init_np).to(dev)
            csteps = CudaSteps(Ssm, 0, cfg.n_train, cfg.m, cfg.sub, cfg.k, dev)
            train_step = lambda: lloyd_sharded(csteps, init_d, tcfg, reduce=args.reduce)
        else:
            train_step = lambda: P.lloyd_iterate_batched(Ssm, init_np, tcfg, return_assignments=False)
        if rank == 0 and "results" in tinfo:
            parity["train"] = train_parity(cfg, dev, tinfo["results"])

        def cs_of(res):
            return P.CodebookSet.from_rowmajor_batch(np.stack([r.centroids for r in res]))

        def step():
            P.encode_dataset_device(X, cs_of(train_step()), plan, out=out)

        Ssm_h = P.pinned_empty(tuple(Ssm.shape), np.float32)
        Ssm_h[:] = Ssm.cpu().numpy()
        train_host = lambda: cs_of(P.lloyd_iterate_batched(Ssm_h, init_np, tcfg, return_assignments=False))
    else:
        def step():
            P.encode_dataset_device(X, cs, plan, out=out)

    # inputs smaller than 2x L2 (c1: 51 MB) would be served from the 126 MB L2 on repeat steps:
    # flush it with an untimed 4x-L2 write between steps and time each step alone
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    in_bytes = rows * cfg.d * cfg.elem_bytes
    flush = torch.empty(4 * l2, dtype=torch.uint8, device=dev) if in_bytes < 2 * l2 else None
    N.call("cspq_encode_stats", None, 1)
    total_ms, step_ms, clk = timed_device_steps(step, steps, warmup, ws, dev, local, flush)
    l2_note = (f"L2 flushed between steps (untimed {4 * l2 >> 20} MB write; input {in_bytes / 2**20:.0f} MB < 2x L2)"
               if flush is not None else f"inputs larger than L2 ({in_bytes / 1e9:.1f} GB/GPU)")
    del flush
    fl = ctypes.c_uint64(0)
    N.call("cspq_encode_stats", ctypes.byref(fl), 1)
    ms_per_step = total_ms / steps
    value = global_rows * steps / (total_ms / 1e3)
    launches_per_step = count_launches(step)

    # encode-kernel-only timing for c2 (its step also trains): the roofline is the encode kernel's
    enc_ms = ms_per_step
    if cfg.name == "c2":
        em, _, _ = timed_device_steps(lambda: P.encode_dataset_device(X, cs, plan, out=out), steps, 1, ws, dev, local)
        enc_ms = em / steps

    e2e = None
    if not args.no_e2e:
        e2e = e2e_record(cfg, args, X, cs, out, ws, dev, steps,
                         train_fn=train_host if cfg.name == "c2" and ws == 1 else None,
                         train_h2d=Ssm_h.nbytes if cfg.name == "c2" and ws == 1 else 0)
        if cfg.name == "c2":
            e2e["scope"] = "train + encode per step"

    rec = None
    if rank == 0:
        rec = {
            "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": ws, "steps": steps,
            "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg, rows, global_rows, ws, scaling), "global_batch": global_rows,
                       "rows_per_gpu": rows, "parallelism": f"rows sharded x{ws} (codebooks broadcast)",
                       "mode": args.mode, "codebook_train_s": tinfo["train_s"],
                       "codebook_training": tinfo["mode"], "l2": l2_note},
            "clocks": clk, "e2e": e2e, "gpu_launches": launches_per_step * steps,
            "gpu_launches_def": "libcspq_b200.so kernel launches per step (host-side launch counter, "
                                "cspq_launch_count, on one extra untimed step) x steps",
            "roofline": roofline_record(cfg, args, rows, enc_ms, dev), "parity": parity,
            "flagged_per_subvector": fl.value / max(1, rows * cfg.m * (steps if cfg.name != "c2" else steps + warmup)),
            "step_ms": step_ms,
        }
        if cfg.name == "c2":
            rec["train"] = {"gpu_s": tinfo["train_s"], "subspaces": cfg.m, "iters": cfg.iters,
                            "sample_rows": cfg.n_train, "encode_ms": enc_ms,
                            "train_ms_in_step": ms_per_step - enc_ms,
                            "encode_only_vec_s": global_rows / (enc_ms / 1e3),
                            "def": "value = N / (training of all subspaces (fp64, tol 0, incl. the final REFERENCE "
                                   "pass, centroids and objective traces copied to the host) + encode of all rows), per step"}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        gen = lambda r: C.generate(cfg, 0, r, dev).cpu().numpy()
        cpu = cpu_baseline_record(cfg, cs.rowmajor, cs.biases, gen, cpu_seconds)
        if cfg.name == "c2":
            Ssm2 = C.subspace_major(C.training_sample(cfg, dev), cfg.m)
            tr = cpu_train_record(cfg, Ssm2, C.lloyd_init(cfg, Ssm2))
            rec["train"]["cpu_baseline"] = tr
            cpu["encode_only_value"] = cpu["value"]
            cpu["value"] = cfg.n / (tr["seconds"] + cfg.n / cpu["encode_only_value"])
            cpu["sample"] += f"; train + encode = N / (training {tr['seconds']:.0f} s + N / encode rate)"
            del Ssm2
        rec["cpu_baseline"] = cpu
    del X, out
    torch.cuda.empty_cache()
    return rec


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2605_25521_b200 import configs as C
    # one rank per GPU; CSPQ_DIST_BACKEND=gloo runs several ranks on fewer GPUs (a functional
    # check of the sharded path on one device -- never a scaling number)
    backend = os.environ.get("CSPQ_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    cfg = C.CONFIGS[args.config]
    line = run_config(cfg, args, ws, rank, local, dev, args.steps, args.warmup, args.cpu_seconds, True)
    if ws == 1 and not args.no_extra:
        extra = {}
        for name in [c for c in args.extra_configs.split(",") if c and c != cfg.name]:
            ecfg = C.CONFIGS[name]
            esteps = max(3, min(args.steps, 20))
            try:
                extra[name] = run_config(ecfg, args, ws, rank, local, dev, esteps, max(3, min(args.warmup, 3)),
                                         min(args.cpu_seconds, 6.0), False)
            except Exception as exc:  # an extra record must never cost the headline line
                extra[name] = {"error": f"{type(exc).__name__}: {exc}"}
            torch.cuda.empty_cache()
        line["extra"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
