"""Time the tensor-core encode under CSPQ_TC_PROBE timing probes (debug only: needs a build
with -DCSPQ_TC_PROBES, e.g. NVFLAGS=-DCSPQ_TC_PROBES scripts/ab_build.sh wt p and CSPQ_LIB_PATH=build/ab/p/libcspq_b200.so;
most probe bits produce garbage codes).  argv: config, comma list of probes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
probes = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
sizes = {"c1": 100_000, "c2": 1_000_000, "c3": 4_000_000, "c4": 16_000_000, "c5": 1_000_000}
cfg = C.CONFIGS[name]; n = sizes[name]
X = C.generate(cfg, 0, n, dev)
rng = np.random.default_rng(0)
rows = X[torch.from_numpy(rng.choice(n, cfg.k, replace=False)).to(dev)].float().cpu().numpy()
rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
plan = P.ExecutionPlan(mode="tensor")
out = P.encode_dataset_device(X, cs, plan)
for pr in probes:
    os.environ["CSPQ_TC_PROBE"] = str(pr)
    P.encode_dataset_device(X, cs, plan, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(os.environ.get("CSPQ_PROBE_REPS", "5"))
    e0.record()
    for _ in range(reps):
        P.encode_dataset_device(X, cs, plan, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    items = (n + 127) // 128 * cfg.m
    cyc = ms * 1e-3 * 1.965e9 * 148 / items
    print(f"{name} probe={pr:4d} {ms:8.3f} ms {n / (ms / 1e3):.3e} vec/s  {cyc:7.0f} cycles/item/SM", flush=True)
