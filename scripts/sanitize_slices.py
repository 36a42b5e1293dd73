"""Small c3/c4 slices of every hot kernel, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck):
  encode_tc_kernel   fix-up mode (encode_dataset_device, mode auto) and mark mode
                     (Lloyd's screened assignment, inside cspq_lloyd_train)
  encode_k256_kernel guarded and exact SIMT modes
  cspq_lloyd_train   all Lloyd kernels (counting-sort scatter, sums, repair, final pass)
  cspq_kmeanspp      k-means++ seeding
Usage: compute-sanitizer --tool <tool> python scripts/sanitize_slices.py [c3|c4] [which]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
which = sys.argv[2] if len(sys.argv) > 2 else "all"
dev = torch.device("cuda", 0)
cfg = C.CONFIGS[name].scaled(n=20_000, n_train=6_000)
X = C.generate(cfg, 0, 3_000, dev)
S = C.training_sample(cfg, dev)[:, : 4 * cfg.sub]  # 4 subspaces
Ssm = C.subspace_major(S, 4).contiguous()
init = C.lloyd_init(cfg, Ssm)
tcfg = P.TrainConfig(k=cfg.k, max_iters=3, tol=0.0)
if which in ("all", "lloyd"):
    res = P.lloyd_iterate_batched(Ssm, init, tcfg)
    print("lloyd ok", res[0].iterations, flush=True)
rng = np.random.default_rng(0)
rm = np.ascontiguousarray(C.lloyd_init(cfg, C.subspace_major(C.training_sample(cfg, dev), cfg.m)).astype(np.float32))
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
modes = {"all": ("tensor", "guarded", "exact"), "tensor": ("tensor",), "simt": ("guarded", "exact")}.get(which, ())
for mode in modes:
    codes = P.encode_dataset_device(X, cs, P.ExecutionPlan(mode=mode))
    torch.cuda.synchronize()
    print("encode", mode, codes.shape, flush=True)
if which in ("all", "kpp"):
    Sh = Ssm.cpu().numpy()
    rngs = [np.random.default_rng(j) for j in range(4)]
    ini = P.training.kmeanspp_init_batched(Ssm, cfg.k, rngs, dev)
    print("kmeans++ ok", ini.shape, flush=True)
torch.cuda.synchronize()
print("done", name, which)
