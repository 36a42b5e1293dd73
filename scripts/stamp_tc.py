"""clock64 stamps of the tensor-core kernel's roles per item (CTA 0): MMA waits / issue, scan
 phases, epilogue.  Needs a -DCSPQ_TC_PROBES -DCSPQ_TC_STAMPS build (scripts/ab_build.sh, CSPQ_LIB_PATH)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CSPQ_TC_PROBE"] = sys.argv[1] if len(sys.argv) > 1 else "16"
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
cfg = C.CONFIGS["c3"]; n = 2_000_000
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
names = ["mma_afull", "mma_tempty", "mma_commit", "obs_tfull", "epi_arrive", "epi_tfull", "epi_release", "epi_done"]
base = st[0, 0]
st = st - base
for i in list(range(0, 12)) + list(range(1000, 1012)):
    print(i, " ".join(f"{names[k]}={st[i,k]:9.0f}" for k in range(8)))
d = np.diff(st[200:1800], axis=0)
print("median per-item deltas:", {names[k]: float(np.median(d[:, k])) for k in range(8)})
print("median epi tfull->release", float(np.median((st[200:1800, 6] - st[200:1800, 5]))), "release->done", float(np.median(st[200:1800, 7] - st[200:1800, 6])))
print("median first-issue(tempty)->obs_tfull", float(np.median(st[200:1800, 3] - st[200:1800, 1])), "obs_tfull->epi_tfull", float(np.median(st[200:1800, 5] - st[200:1800, 3])), "epi_tfull->arrive", float(np.median(st[200:1800, 4] - st[200:1800, 5])), "arrive(it)->mma_tempty(it+2)", float(np.median(st[202:1800, 1] - st[200:1798, 4])))
print("median mma tempty wait (tempty - afull)", float(np.median(st[200:1800, 1] - st[200:1800, 0])), "commit->epi tfull", float(np.median(st[200:1800, 5] - st[200:1800, 2])))
