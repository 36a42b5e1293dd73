"""Flag rate of the tensor-core screen inside the Lloyd training (c2/c3/c4 samples): the share of
(point, subspace) pairs that take the float64 settle scan."""
import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import torch, paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C, _native as N
dev = torch.device("cuda", 0)
for name in ["c2", "c3", "c4"]:
    cfg = C.CONFIGS[name]
    S = C.training_sample(cfg, dev); Ssm = C.subspace_major(S, cfg.m); init = C.lloyd_init(cfg, Ssm)
    N.call("cspq_encode_stats", None, 1)
    P.lloyd_iterate_batched(Ssm, init, P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0))
    fl = ctypes.c_uint64(0); N.call("cspq_encode_stats", ctypes.byref(fl), 1)
    tot = cfg.m * cfg.n_train * cfg.iters
    print(name, "flag rate", fl.value / tot, "flagged", fl.value)
