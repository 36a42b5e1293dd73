"""Time the batched GPU Lloyd (lloyd_iterate_batched) on the configs' training samples."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c3", "c4"]):
    cfg = C.CONFIGS[name]
    S = C.training_sample(cfg, dev)
    Ssm = C.subspace_major(S, cfg.m)
    init = C.lloyd_init(cfg, Ssm)
    tc = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
    P.lloyd_iterate_batched(Ssm, init, tc)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.lloyd_iterate_batched(Ssm, init, tc)
    dt = time.perf_counter() - t0
    flops = 2.0 * cfg.m * cfg.n_train * cfg.k * cfg.sub * cfg.iters
    print(f"{name}: m={cfg.m} n={cfg.n_train} iters={cfg.iters}: {dt * 1e3:.1f} ms  "
          f"(assign {flops / dt / 1e12:.2f} TFLOP/s fp64 equiv)  obj0={res[0].objectives[-1]:.6g}", flush=True)
