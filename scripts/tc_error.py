"""Measure |S_tc - s_oracle| / W on winners across data regimes (W = max|b| + ||x|| max||c||)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from oracle import oracle as O
from paper_2605_25521_b200 import configs as C
def run(X, rm, label):
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(rm.shape[0])])
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    b = torch.empty((X.shape[0], cs.m), dtype=torch.float32, device="cuda")
    codes = P.encode_dataset_device(Xd, cs, P.ExecutionPlan(mode="tensor"), best=b).cpu().numpy()
    want, wbest = O.encode(X, cs.rowmajor, cs.biases, O.VARIANT_REFORM, want_best=True)
    same = codes == want
    sub = cs.sub_dim
    xs = X.astype(np.float64).reshape(X.shape[0], cs.m, sub)
    nrm = np.sqrt((xs ** 2).sum(-1))
    bmax = np.abs(cs.biases.astype(np.float64)).max(axis=1)
    cmax = np.sqrt((cs.rowmajor.astype(np.float64) ** 2).sum(-1)).max(axis=1)
    W = bmax[None, :] + nrm * cmax[None, :]
    # tighter per-row scale: |b_l*| + sum_t |x_t c_l*t| for the winner l*
    err = np.abs(b.cpu().numpy().astype(np.float64) - wbest.astype(np.float64))[same]
    r = err / W[same]
    print(f"{label:28s} max err/W {r.max():.3e}  p99.99 {np.quantile(r, 0.9999):.3e}  mean {r.mean():.3e}  (bound 8.9e-6)")
rng = np.random.default_rng(0)
dev = torch.device("cuda", 0)
for name in ["c1", "c2", "c3", "c4", "c5"]:
    cfg = C.CONFIGS[name]
    Xg = C.generate(cfg, 0, 100_000, dev)
    X = Xg.cpu().numpy().astype(np.float32)
    rows = X[rng.choice(X.shape[0], 256, replace=False)]
    rm = np.ascontiguousarray(rows.reshape(256, cfg.m, cfg.sub).transpose(1, 0, 2))
    run(X, rm, name)
for scale in (1.0, 1e4, 1e-4):
    X = (rng.standard_normal((50_000, 64)) * scale).astype(np.float32)
    rm = (rng.standard_normal((8, 256, 8)) * scale).astype(np.float32)
    run(X, rm, f"normal scale {scale:g}")
# heavy cancellation: x nearly orthogonal to large centroids with huge biases
X = (rng.standard_normal((50_000, 64)) * 100).astype(np.float32)
rm = (rng.standard_normal((8, 256, 8)) * 100 + 1000).astype(np.float32)
run(X, rm, "offset centroids")
