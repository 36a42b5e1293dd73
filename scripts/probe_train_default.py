"""Time the reference-default training path (train_all_codebooks: per-subspace sampling,
k-means++ seeding, Lloyd with tol stop) on c3-shaped data."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
cfg = C.CONFIGS["c3"]
X = C.generate(cfg, 0, 200_000, torch.device("cuda", 0)).cpu().numpy()
ds = P.VectorDataset(data=X)
params, tc = P.PQParams(d=cfg.d, m=cfg.m, k=256), P.TrainConfig(k=256, seed=0)
P.train_all_codebooks(P.VectorDataset(data=X[:20000]), params, P.TrainConfig(k=256, seed=0, max_iters=2))  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
cbs, reps = P.train_all_codebooks_report(ds, params, tc)
dt = time.perf_counter() - t0
print(f"train_all_codebooks c3-shaped 200k x 768, m=96, k=256 (k-means++ + Lloyd, tol 1e-4): {dt:.2f} s; "
      f"iterations min/median/max {min(r.iterations for r in reps)}/{int(np.median([r.iterations for r in reps]))}/"
      f"{max(r.iterations for r in reps)}", flush=True)
# phase split
from paper_2605_25521_b200.training import _subspace_rngs, _sample, _validate_points, kmeanspp_init_batched, lloyd_iterate_batched
rngs = _subspace_rngs(0, cfg.m)
t0 = time.perf_counter()
sampled = []
for j, r in enumerate(rngs):
    s = np.asarray(_sample(X[:, j * 8:(j + 1) * 8], tc.resolved_cap(), r), dtype=np.float64)
    _validate_points(s, 256)
    sampled.append(s)
t1 = time.perf_counter()
init = kmeanspp_init_batched(sampled, 256, rngs)
t2 = time.perf_counter()
lloyd_iterate_batched(sampled, init, tc)
t3 = time.perf_counter()
print(f"phases: sample+validate {t1 - t0:.2f} s, k-means++ {t2 - t1:.2f} s, Lloyd {t3 - t2:.2f} s", flush=True)
