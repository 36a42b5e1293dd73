"""Time the batched GPU k-means++ seeding."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200.training import _subspace_rngs, kmeanspp_init_batched
rng = np.random.default_rng(0)
pts = [rng.standard_normal((65536, 8)) for _ in range(96)]
kmeanspp_init_batched(pts, 32, _subspace_rngs(0, 96))
torch.cuda.synchronize()
t0 = time.perf_counter()
kmeanspp_init_batched(pts, 64, _subspace_rngs(0, 96))
print("kpp k=64:", time.perf_counter() - t0)
