"""encode_dataset on a pageable numpy array (the common call) vs pinned host buffers."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
cfg = C.CONFIGS["c3"]
n = 2_000_000
Xd = C.generate(cfg, 0, n, torch.device("cuda", 0))
X = Xd.cpu().numpy().copy()                      # pageable
rng = np.random.default_rng(0)
rm = (rng.standard_normal((cfg.m, 256, cfg.sub)) * 0.2).astype(np.float32)
cbs = [P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)]
cs = P.CodebookSet.from_codebooks(cbs)
P.encode_dataset(X[:100000], cs)
for label, arr in (("pageable", X), ("pinned", None)):
    if arr is None:
        arr = P.pinned_empty(X.shape, np.float32)
        arr[:] = X
    for plan in (P.ExecutionPlan(), P.ExecutionPlan(), P.ExecutionPlan(streams=4), P.ExecutionPlan(streams=6)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        codes = P.encode_dataset(arr, cs, plan).codes
        dt = time.perf_counter() - t0
        print(f"{label:8s} batch={plan.resolved_batch_rows():7d} streams={plan.streams}: {n / dt / 1e6:6.2f} M vec/s "
              f"({n * cfg.d * 4 / dt / 1e9:5.1f} GB/s)", flush=True)
