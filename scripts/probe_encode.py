"""Quick timing probe of the encode kernel modes on config-shaped data."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C

dev = torch.device("cuda", 0)
for name, n in (("c3", 2_000_000), ("c4", 8_000_000), ("c1", 100_000)):
    cfg = C.CONFIGS[name]
    X = C.generate(cfg, 0, n, dev)
    rng = np.random.default_rng(0)
    idx = rng.choice(n, cfg.k, replace=False)
    rows = X[torch.from_numpy(idx).to(dev)].float().cpu().numpy()
    rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
    for mode in ("exact", "guarded"):
        plan = P.ExecutionPlan(mode=mode)
        import ctypes
        from paper_2605_25521_b200 import _native as N
        N.call("cspq_encode_stats", None, 1)
        out = P.encode_dataset_device(X, cs, plan)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            P.encode_dataset_device(X, cs, plan, out=out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        vps = n / (ms / 1e3)
        tf = vps * cfg.flops_per_vec() / 1e12
        import ctypes
        from paper_2605_25521_b200 import _native as N
        fl = ctypes.c_uint64(0)
        N.call("cspq_encode_stats", ctypes.byref(fl), 1)
        print(f"{name} n={n} mode={mode}: {ms:.2f} ms  {vps:.3e} vec/s  {tf:.1f} TFLOP/s ({tf/74.45*100:.1f}% of 74.45) flagged/subvec={fl.value/((reps+1)*n*cfg.m):.2e}", flush=True)
