"""Time tensor-core vs FFMA encode on config-shaped data."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C, _native as N
dev = torch.device("cuda", 0)
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c4", "c1", "c2", "c5"]
sizes = {"c1": 100_000, "c2": 1_000_000, "c3": 4_000_000, "c4": 16_000_000, "c5": 1_000_000}
for name in names:
    cfg = C.CONFIGS[name]; n = sizes[name]
    X = C.generate(cfg, 0, n, dev)
    rng = np.random.default_rng(0)
    rows = X[torch.from_numpy(rng.choice(n, cfg.k, replace=False)).to(dev)].float().cpu().numpy()
    rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
    ref = None
    for mode in ("tensor", "guarded"):
        plan = P.ExecutionPlan(mode=mode)
        out = P.encode_dataset_device(X, cs, plan)
        torch.cuda.synchronize()
        ref = out.clone() if ref is None else ref
        same = bool(torch.equal(out, ref))
        N.call("cspq_encode_stats", None, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            P.encode_dataset_device(X, cs, plan, out=out)
        e1.record(); torch.cuda.synchronize()
        fl = ctypes.c_uint64(0); N.call("cspq_encode_stats", ctypes.byref(fl), 1)
        ms = e0.elapsed_time(e1) / reps
        vps = n / (ms / 1e3); tf = vps * cfg.flops_per_vec() / 1e12
        gbs = vps * cfg.bytes_per_vec() / 1e9
        print(f"{name} n={n} {mode:8s} {ms:8.3f} ms {vps:.3e} vec/s {tf:6.1f} TF/s ({tf/74.45*100:5.1f}% fp32) {gbs:7.1f} GB/s flag={fl.value/(reps*n*cfg.m):.1e} same={same}", flush=True)
