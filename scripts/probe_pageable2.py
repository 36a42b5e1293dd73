"""Repeated timing of encode_dataset on a pageable numpy array (staged through the pinned ring); CSPQ_HOST_COPY_NT=0/1
selects memcpy / non-temporal staging copies (read once per process)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
cfg = C.CONFIGS["c3"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
Xd = C.generate(cfg, 0, n, torch.device("cuda", 0))
X = Xd.cpu().numpy().copy()
rng = np.random.default_rng(0)
rm = (rng.standard_normal((cfg.m, 256, cfg.sub)) * 0.2).astype(np.float32)
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
P.encode_dataset(X[:100000], cs)
r = []
for _ in range(6):
    t0 = time.perf_counter()
    P.encode_dataset(X, cs)
    r.append(n * cfg.d * 4 / (time.perf_counter() - t0) / 1e9)
print("NT", os.environ.get("CSPQ_HOST_COPY_NT", "1"), " ".join(f"{v:5.1f}" for v in r), "GB/s of rows")
