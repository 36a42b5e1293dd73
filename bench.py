#!/usr/bin/env python
"""bench.py -- PQ-encoded vectors/s on B200 (BASELINE.json metric).

Workload (default): BASELINE config 3 -- N = 10,000,000 unit-normalised
float32 rows per GPU, D = 768, M = 96 subspaces (d_sub = 8), K = 256,
codebooks from 10 Lloyd iterations (GPU, fp64) on a 200,000-row seeded
sample, trained on rank 0 and broadcast over NCCL.  A "step" is one encode
pass of the whole shard (one fused kernel launch).  Weak scaling: every rank
encodes its own 10M-row shard of one seeded dataset (rows r*N .. (r+1)*N).

Launch: python bench.py [--gpus N --steps K --warmup W]
        torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)
        python bench.py --impl reference ...   (the CPU oracle, host cores)

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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--rows", type=int, default=0, help="rows per rank (0 = the config's N)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    p.add_argument("--mode", default="auto", choices=["auto", "exact", "guarded"])
    p.add_argument("--e2e-rows", type=int, default=0,
                   help="rows per rank through the host API (0 = max(2M, 6 GB of rows), or the whole config for c5)")
    p.add_argument("--streams", type=int, default=0, help="host pipeline streams (0 = 3, or 6 for c5)")
    p.add_argument("--e2e-batch", type=int, default=0, help="host pipeline batch rows (0 = max(131072 rows, 256 MB) capped at a quarter of the sample, or 4096 for c5)")
    p.add_argument("--train", choices=["auto", "sharded", "rank0"], default="auto",
                   help="codebook training: row-sharded Lloyd with one all-reduce per iteration (auto: when N > 1), "
                        "or the fused single-GPU cspq_lloyd_train on rank 0 + broadcast")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_desc(cfg, rows_per_rank, ws, scaling):
    return (f"{cfg.name}: {'u8' if cfg.dtype == 'u8' else 'f32'} rows D={cfg.d}, M={cfg.m} (d_sub={cfg.sub}), "
            f"K={cfg.k}, {rows_per_rank:,} rows/GPU ({scaling} scaling), codebooks: "
            + (f"{cfg.iters} Lloyd iters on a {cfg.n_train:,}-row sample" if cfg.codebook == "lloyd"
               else "256 distinct data subvectors per subspace")
            + ("; timed steps encode, the training is timed once in train.* (train_plus_encode_vec_s: both)"
               if cfg.name == "c2" else ""))


def oracle_codebooks(cfg, dev):
    """Codebooks for the reference arm: the config's Lloyd initial points
    (no GPU compute -- only the seeded data generator)."""
    import numpy as np
    from paper_2605_25521_b200 import configs as C
    if cfg.codebook == "sampled":  # c1: distinct data subvectors, as the B200 arm uses
        rm = np.ascontiguousarray(C.sampled_codebooks(cfg, C.generate(cfg, 0, cfg.n, dev).cpu().numpy()))
    else:
        S = C.training_sample(cfg, dev)
        rm = np.ascontiguousarray(C.lloyd_init(cfg, C.subspace_major(S, cfg.m)).astype(np.float32))
    from oracle.oracle import compute_biases
    return rm, compute_biases(rm)


def cpu_oracle_rate(cfg, dev, rm, bs, seconds, rows_hint=50_000):
    """Time the CPU oracle (strict-fp32 restatement of the reference's
    encoder, all host threads) on bounded samples of the workload's rows."""
    import numpy as np
    from oracle import oracle as O
    from paper_2605_25521_b200 import configs as C
    cores = os.cpu_count() or 1
    warm = C.generate(cfg, 0, min(rows_hint, 20_000), dev).cpu().numpy()
    O.encode(warm, rm, bs, O.VARIANT_REFORM, threads=cores)
    t0 = time.perf_counter()
    O.encode(warm, rm, bs, O.VARIANT_REFORM, threads=cores)
    per_row = (time.perf_counter() - t0) / warm.shape[0]
    rows = int(max(10_000, min(cfg.n, seconds / max(per_row, 1e-9))))
    X = C.generate(cfg, 0, rows, dev).cpu().numpy()
    t0 = time.perf_counter()
    O.encode(X, rm, bs, O.VARIANT_REFORM, threads=cores)
    dt = time.perf_counter() - t0
    return rows / dt, rows, dt, cores


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle of the reference's encoder on the
    host cores, same config/metric; rank 0 only."""
    if rank != 0:
        return
    import numpy as np
    import torch
    from paper_2605_25521_b200 import configs as C
    from oracle import oracle as O
    cfg = C.CONFIGS[args.config]
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    rm, bs = oracle_codebooks(cfg, dev)
    cores = os.cpu_count() or 1
    rate, rows, _, _ = cpu_oracle_rate(cfg, dev, rm, bs, 3.0)
    X = C.generate(cfg, 0, rows, dev).cpu().numpy()
    for _ in range(args.warmup):
        O.encode(X, rm, bs, O.VARIANT_REFORM, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.encode(X, rm, bs, O.VARIANT_REFORM, threads=cores)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = rows / (ms / 1e3)
    sample = f"{rows:,} rows of {cfg.name} per step (oracle/pq_oracle.c, strict fp32, {cores} threads)"
    line = {
        "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_desc(cfg, rows, 1, args.scaling), "rows_per_step": rows},
        "cpu_baseline": {"value": value, "unit": "vectors/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "vectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_25521_b200 as P
    from paper_2605_25521_b200 import _native as N
    from paper_2605_25521_b200 import configs as C
    from paper_2605_25521_b200.telemetry import ClockSampler

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = C.CONFIGS[args.config]
    rows = args.rows or cfg.n
    if args.scaling == "strong":
        rows = rows // ws
    begin = rank * rows

    # ---- data (device-resident, seeded, chunk-deterministic) ----
    X = C.generate(cfg, begin, begin + rows, dev)

    # ---- codebooks: GPU Lloyd on rank 0, NCCL broadcast ----
    rm = torch.empty((cfg.m, cfg.k, cfg.sub), dtype=torch.float32, device=dev)
    train_s = None
    sharded = args.train == "sharded" or (args.train == "auto" and ws > 1)
    train_mode = ("sampled codebooks" if cfg.codebook == "sampled" else "fused cspq_lloyd_train") + \
        (" on rank 0 + NCCL broadcast" if ws > 1 else "")
    if cfg.codebook == "lloyd" and sharded:
        # north_star scheme: every rank assigns its row shard of the training sample and one
        # NCCL all-reduce per iteration combines (counts, sums, objective terms)
        from paper_2605_25521_b200.distributed import CudaSteps, lloyd_sharded
        S = C.training_sample(cfg, dev)
        Ssm = C.subspace_major(S, cfg.m).contiguous()
        init = torch.from_numpy(C.lloyd_init(cfg, Ssm)).to(dev)
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = lloyd_sharded(CudaSteps(Ssm, 0, cfg.n_train, cfg.m, cfg.sub, cfg.k, dev), init,
                            P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0), reduce="allreduce")
        train_s = time.perf_counter() - t0
        rm.copy_(torch.from_numpy(np.stack([r.centroids for r in res])))
        train_mode = (f"row-sharded x{ws}, one NCCL all-reduce per iteration" if ws > 1
                      else "row-sharded driver at world size 1 (no collective)")
        del S, Ssm
    elif rank == 0:
        if cfg.codebook == "sampled":
            Xh = C.generate(cfg, 0, cfg.n, dev).cpu().numpy()
            rm.copy_(torch.from_numpy(C.sampled_codebooks(cfg, Xh)))
        else:
            S = C.training_sample(cfg, dev)
            Ssm = C.subspace_major(S, cfg.m)
            init = C.lloyd_init(cfg, Ssm)
            P.lloyd_iterate_batched(Ssm, init, P.TrainConfig(k=cfg.k, max_iters=1, tol=0.0))  # untimed warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = P.lloyd_iterate_batched(Ssm, init, P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0))
            train_s = time.perf_counter() - t0
            rm.copy_(torch.from_numpy(np.stack([r.centroids for r in res])))
            del S, Ssm
    if ws > 1:
        dist.broadcast(rm, src=0)
    rmh = rm.cpu().numpy()
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rmh[j]) for j in range(cfg.m)])
    plan = P.ExecutionPlan(mode=args.mode)
    out = P.encode_dataset_device(X, cs, plan)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    # ---- parity spot-check vs the oracle (rank 0, sampled rows) ----
    parity = None
    if rank == 0:
        from oracle import oracle as O
        rng = np.random.default_rng(123)
        idx = np.sort(rng.choice(rows, min(rows, 20_000), replace=False))
        ti = torch.from_numpy(idx).to(dev)
        want = O.encode(X[ti].cpu().numpy(), cs.rowmajor, cs.biases, O.VARIANT_REFORM)
        got = out[ti].cpu().numpy()
        parity = {"rows_checked": int(idx.shape[0]), "code_mismatches": int((got != want).sum())}

    # ---- device-resident timed region ----
    # inputs smaller than 2x L2 (c1: 51 MB) would be served from the 126 MB L2 on repeat
    # steps: flush it with an untimed 4x-L2 write between steps and time each step alone
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    in_bytes = rows * cfg.d * cfg.elem_bytes
    flush = torch.empty(4 * l2, dtype=torch.uint8, device=dev) if in_bytes < 2 * l2 else None
    for _ in range(args.warmup):
        P.encode_dataset_device(X, cs, plan, out=out)
    N.call("cspq_encode_stats", None, 1)
    clocks = ClockSampler(local).start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        if flush is not None:
            flush.fill_(s & 0xff)
        ev[2 * s].record(stream)
        P.encode_dataset_device(X, cs, plan, out=out)
        ev[2 * s + 1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [ev[2 * s].elapsed_time(ev[2 * s + 1]) for s in range(args.steps)]
    total_ms = sum(step_ms) if flush is not None else ev[0].elapsed_time(ev[-1])
    l2_note = (f"L2 flushed between steps (untimed {4 * l2 >> 20} MB write; input {in_bytes / 2**20:.0f} MB < 2x L2)"
               if flush is not None else f"inputs larger than L2 ({in_bytes / 1e9:.1f} GB/GPU)")
    del flush
    fl = ctypes.c_uint64(0)
    N.call("cspq_encode_stats", ctypes.byref(fl), 1)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = rows * ws * args.steps / (total_ms / 1e3)

    # ---- end-to-end through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        # c5 is the streaming config: the reference's 4096-row batches from pinned host memory,
        # whole dataset per step, with per-batch H2D -> encode -> D2H latency from device events
        # sized in bytes, so short rows (c4: 128 B) get batches and samples as large as long ones:
        # ~6 GB of rows per step and batches of >= 128K rows and >= 256 MB (c3: 2M rows, 128K-row
        # batches -- 128K..1M rows all saturate PCIe at 54-55 GB/s; c4: 47M rows, 2M-row batches)
        row_bytes = cfg.d * cfg.elem_bytes
        ne = min(args.e2e_rows or (cfg.n if cfg.batch else max(2_000_000, (6 << 30) // row_bytes)), rows)
        batch_rows = cfg.batch or args.e2e_batch or max(1 << 17, (256 << 20) // row_bytes)
        if not (cfg.batch or args.e2e_batch):
            # at least 4 batches so encode and D2H overlap the next H2D (c1's 100K rows: 4 x 25K)
            batch_rows = min(batch_rows, max(1 << 14, -(-ne // 4)))
        Xh = P.pinned_empty((ne, cfg.d), np.uint8 if cfg.dtype == "u8" else np.float32)
        Xh[:] = X[:ne].cpu().numpy()
        codes_h = P.pinned_empty((ne, cfg.m), np.uint8)
        eplan = P.ExecutionPlan(mode=args.mode, batch_rows=batch_rows, streams=args.streams or (6 if cfg.batch else 3))
        nb = (ne + batch_rows - 1) // batch_rows
        bms = np.zeros(nb, np.float64)
        P.encode_dataset_host(Xh, cs, eplan, out=codes_h)  # warm the pipeline
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        lat = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            P.encode_dataset_host(Xh, cs, eplan, out=codes_h, batch_ms=bms)
            lat.append(bms.copy())
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e_val = ne * ws * args.steps / float(el.item())
        assert np.array_equal(codes_h[:4096], out[:4096].cpu().numpy()), "e2e codes differ from device codes"
        lat = np.concatenate(lat)
        e2e = {"value": e2e_val, "unit": "vectors/s", "h2d_bytes_per_step": int(ne * cfg.d * cfg.elem_bytes) * ws,
               "d2h_bytes_per_step": int(ne * cfg.m) * ws, "rows_per_gpu": ne, "batch_rows": batch_rows,
               "streams": eplan.streams,
               "batch_latency_ms": {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                                    "batches": int(lat.shape[0]),
                                    "def": f"device events: H2D start -> D2H end of one batch ({eplan.streams} batches in flight)"},
               "h2d_GBps": ne * cfg.d * cfg.elem_bytes * args.steps / float(el.item()) / 1e9,
               "path": "encode_dataset_host (pinned numpy -> cspq_encode_host: multi-stream H2D/encode/D2H pipeline)"}

    # ---- roofline of the encode kernel ----
    flops_launch = rows * cfg.flops_per_vec()
    achieved = flops_launch / (ms_per_step / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "encode_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            key = cfg.name + ("_tc" if args.mode in ("auto", "tensor") else "")
            bpr = tj.get(key, {}).get("dram_bytes_per_row")
            traffic = None if bpr is None else int(bpr * rows)
        except Exception:
            traffic = None
    tc = args.mode in ("auto", "tensor") and cfg.k == 256 and cfg.sub in (4, 8)
    tf32_peak = None
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            tf32_peak = json.load(open(mp))["bf16_tflops"] / 2.0  # dense tf32 = half of dense bf16
        except Exception:
            tf32_peak = None
    if tf32_peak is None:
        tf32_peak = 1590.0 / 2.0  # B200_PROFILING.md fallback bf16 burst / 2
    k_eff = 32 if cfg.sub == 8 else 16  # tf32 MMA K per (row, subspace): 3xTF32 split + bias + pad
    roofline = {"bound": "fp32", "achieved": achieved, "peak": FP32_NOMINAL_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP32_NOMINAL_TFLOPS, "traffic": traffic,
                "kernel": ("encode_tc_kernel (tcgen05 3xTF32 + exact epilogue)" if tc else
                           "encode_k256_kernel (" + ("exact" if args.mode == "exact" else "guarded FFMA") + ")"),
                "peak_source": "north_star roofline = the slower of FP32 FFMA and tensor peaks: nominal FP32 "
                               "148 SMs x 128 lanes x 2 flop x 1.965 GHz (no FP32 entry in MEASURED_PEAKS.json)",
                "algorithmic_flops_per_row": cfg.flops_per_vec(),
                "algorithmic_bytes_per_row": cfg.bytes_per_vec(),
                "hbm_frac": (rows * cfg.bytes_per_vec() / (ms_per_step / 1e3) / 1e9) / 6547.8}
    if tc:
        roofline["tensor"] = {
            "peak_tf32_tflops": tf32_peak, "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2",
            "algorithmic_frac": achieved / tf32_peak,
            "executed_tensor_tflops": achieved * (k_eff / cfg.sub),
            "executed_frac": achieved * (k_eff / cfg.sub) / tf32_peak,
            "note": f"the MMA executes K={k_eff} tf32 per (row, subspace) for {cfg.sub} useful MACs "
                    "(hi/lo split + folded bias); the epilogue's min/max on the half-rate ALU pipe is the binding unit",
        }
        # the binding unit: an exact argmin with an exact runner-up over K scores needs two min
        # trees (block and class minima) -- K three-input min lane-operations per (row, subspace) --
        # on the ALU pipe (16 lanes / clk / SMSP, scripts/micro/mnmx_peak.cu)
        alu_peak = torch.cuda.get_device_properties(dev).multi_processor_count * 4 * 16 * 1.965e9
        alu_ops = rows * cfg.m * cfg.k / (ms_per_step / 1e3)
        roofline["alu"] = {
            "algorithmic_min_lane_ops_per_row": cfg.m * cfg.k, "achieved_lane_ops_per_s": alu_ops,
            "peak_lane_ops_per_s": alu_peak, "frac": alu_ops / alu_peak,
            "note": "FMNMX3 lane-ops of the two min trees only; ncu shows the ALU pipe ~56 % busy in total "
                    "(the rest: predicates, loop and address arithmetic), profiles/r1_ncu_full_encode_c3_tc.json",
        }
    # ---- c2's timed scope is train + encode: report the GPU Lloyd beside the encode ----
    train = None
    if rank == 0 and cfg.codebook == "lloyd" and cfg.name == "c2":
        enc_s = ms_per_step / 1e3
        train = {"gpu_s": train_s, "subspaces": cfg.m, "iters": cfg.iters, "sample_rows": cfg.n_train,
                 "train_plus_encode_vec_s": rows / (train_s + enc_s),
                 "mode": train_mode,
                 "def": "wall time of the codebook training (all subspaces, fp64, tol=0) incl. the final "
                        "REFERENCE pass and host transfer of the results, after an untimed 1-iteration warm-up"}
        if ws == 1 and not args.no_cpu_baseline:
            from oracle import oracle as O
            S = C.training_sample(cfg, dev)
            Ssm = C.subspace_major(S, cfg.m)
            init = C.lloyd_init(cfg, Ssm)
            p0 = Ssm[0].double().cpu().numpy()
            t0 = time.perf_counter()
            O.lloyd(p0, init[0], cfg.iters, 0.0)
            one = time.perf_counter() - t0
            train["cpu_baseline"] = {"seconds": one * cfg.m, "kind": "port", "cores": os.cpu_count() or 1,
                                     "sample": f"oracle.lloyd on subspace 0 ({cfg.n_train:,} x {cfg.sub} fp64, "
                                               f"{cfg.iters} iters) in {one:.2f} s, x {cfg.m} subspaces"}
            del S, Ssm
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, crow, cdt, cores = cpu_oracle_rate(cfg, dev, cs.rowmajor, cs.biases, args.cpu_seconds)
        cpu = {"value": rate, "unit": "vectors/s", "cores": cores, "kind": "port",
               "sample": f"{crow:,} rows of {cfg.name} in {cdt:.1f} s (oracle/pq_oracle.c strict-fp32 restatement of "
                         f"the reference encoder, OpenMP over all host threads)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "vectors/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg, rows, ws, args.scaling), "global_batch": rows * ws,
                       "rows_per_gpu": rows, "parallelism": f"rows sharded x{ws} (codebooks NCCL-broadcast)",
                       "mode": args.mode, "codebook_train_s": train_s, "codebook_training": train_mode,
                       "l2": l2_note},
            "clocks": clk, "e2e": e2e, "gpu_launches": args.steps, "roofline": roofline, "cpu_baseline": cpu,
            "parity": parity, "flagged_per_subvector": fl.value / max(1, rows * cfg.m * args.steps),
            "step_ms": step_ms,
        }
        if train is not None:
            line["train"] = train
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
