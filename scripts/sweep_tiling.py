"""Sweep the fast-encode tiling on config-shaped data (timing + flag rate)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C, _native as N
dev = torch.device("cuda", 0)
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c4"]
sizes = {"c1": 100_000, "c2": 1_000_000, "c3": 2_000_000, "c4": 8_000_000, "c5": 1_000_000}
for name in names:
    cfg = C.CONFIGS[name]; n = sizes[name]
    X = C.generate(cfg, 0, n, dev)
    rng = np.random.default_rng(0)
    rows = X[torch.from_numpy(rng.choice(n, cfg.k, replace=False)).to(dev)].float().cpu().numpy()
    rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
    ref = None
    for tiling in range(4):
        N.call("cspq_encode_set_tiling", tiling)
        for mode in ("guarded", "exact"):
            plan = P.ExecutionPlan(mode=mode)
            out = P.encode_dataset_device(X, cs, plan)
            torch.cuda.synchronize()
            ref = out.clone() if ref is None else ref
            same = bool(torch.equal(out, ref))
            N.call("cspq_encode_stats", None, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                P.encode_dataset_device(X, cs, plan, out=out)
            e1.record(); torch.cuda.synchronize()
            fl = ctypes.c_uint64(0); N.call("cspq_encode_stats", ctypes.byref(fl), 1)
            ms = e0.elapsed_time(e1) / reps
            vps = n / (ms / 1e3); tf = vps * cfg.flops_per_vec() / 1e12
            print(f"{name} tiling={tiling} {mode:8s} {ms:7.2f} ms {vps:.3e} vec/s {tf:5.1f} TF/s ({tf/74.45*100:4.1f}%) flag={fl.value/(reps*n*cfg.m):.1e} same={same}", flush=True)
    N.call("cspq_encode_set_tiling", 3)
