"""clock64 stamps of the v2 (team) tensor-core kernel per item (CTA 0).  Needs a
-DCSPQ_TC_PROBES -DCSPQ_TC_STAMPS build (scripts/ab_build.sh) and CSPQ_TC_KERNEL=2."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CSPQ_TC_PROBE"] = "16"
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
cfg = C.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]; n = 2_000_000
X = C.generate(cfg, 0, n, dev)
rng = np.random.default_rng(0)
rows = X[torch.from_numpy(rng.choice(n, cfg.k, replace=False)).to(dev)].float().cpu().numpy()
rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
best = torch.zeros((n, cfg.m), dtype=torch.float32, device=dev)
for _ in range(2):
    best.zero_()
    P.encode_dataset_device(X, cs, P.ExecutionPlan(mode="tensor"), best=best)
torch.cuda.synchronize()
st = best.view(torch.int64).flatten()[:2048 * 8].cpu().numpy().reshape(2048, 8).astype(np.float64)
names = ["mma_afull", "mma_tempty", "mma_commit", "h0_tfull", "h0_release", "h0_bar", "h0_done", "h1_tfull"]
st = st - st[0, 0]
for i in list(range(1000, 1016)):
    print(i, " ".join(f"{names[k]}={st[i,k]:9.0f}" for k in range(8)))
sl = st[200:1800]
print("median per-item deltas:", {names[k]: float(np.median(np.diff(sl[:, k]))) for k in range(8)})
def med(a, b): return float(np.median(sl[:, b] - sl[:, a]))
print("commit->h0_tfull", med(2, 3), "h0_tfull->release", med(3, 4), "release->bar", med(4, 5), "bar->done", med(5, 6),
      "h1 tfull - h0 tfull", med(3, 7), "afull->tempty", med(0, 1), "tempty->commit", med(1, 2))
