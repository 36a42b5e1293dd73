"""Encode the same config-shaped rows with the library named by CSPQ_LIB_PATH and save / compare the
codes (A/B check of kernel variants: python scripts/cmp_variants.py c3 2000000 save|cmp /tmp/codes.npy)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
name, n, mode, path = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
dev = torch.device("cuda", 0)
cfg = C.CONFIGS[name]
X = C.generate(cfg, 0, n, dev)
rng = np.random.default_rng(0)
rows = X[torch.from_numpy(rng.choice(n, cfg.k, replace=False)).to(dev)].float().cpu().numpy()
rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
outs = [P.encode_dataset_device(X, cs, P.ExecutionPlan(mode="tensor")).cpu().numpy() for _ in range(3)]
assert all((o == outs[0]).all() for o in outs), "non-deterministic codes"
if mode == "save":
    np.save(path, outs[0]); print("saved", outs[0].shape)
else:
    ref = np.load(path); bad = int((ref != outs[0]).sum()); print("mismatches vs saved:", bad, "of", ref.size); assert bad == 0
