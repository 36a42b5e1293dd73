import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
cfg = C.CONFIGS["c2"]
S = C.training_sample(cfg, dev); Ssm = C.subspace_major(S, cfg.m); init = C.lloyd_init(cfg, Ssm)
tc = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
P.lloyd_iterate_batched(Ssm, init, tc, return_assignments=False)
torch.cuda.synchronize()
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    P.lloyd_iterate_batched(Ssm, init, tc, return_assignments=False)
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"wall {1e3*(t1-t0):.2f} ms, events {e0.elapsed_time(e1):.2f} ms")
