"""Phase timings of the reference-default training path (train_all_codebooks) on c3-shaped data."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C, training as T
from paper_2605_25521_b200._device import device, to_device
cfg = C.CONFIGS["c3"]
X = C.generate(cfg, 0, 200_000, torch.device("cuda", 0)).cpu().numpy()
tc = P.TrainConfig(k=256, seed=0)
P.train_all_codebooks(P.VectorDataset(data=X[:20000]), P.PQParams(d=cfg.d, m=cfg.m, k=256), P.TrainConfig(k=256, seed=0, max_iters=2))
torch.cuda.synchronize()
t = [time.perf_counter()]
rngs = T._subspace_rngs(0, cfg.m)
pts = [X[:, j * 8:(j + 1) * 8] for j in range(cfg.m)]
samples = [T._sample(p, tc.resolved_cap(), r) for p, r in zip(pts, rngs)]; t.append(time.perf_counter())
s64 = [np.asarray(s, dtype=np.float64) for s in samples]; t.append(time.perf_counter())
for s in s64: T._validate_points(s, 256)
t.append(time.perf_counter())
Pst, _ = T._stack_points(s64); t.append(time.perf_counter())
Pd = to_device(Pst, device()); torch.cuda.synchronize(); t.append(time.perf_counter())
init = T.kmeanspp_init_batched(Pd, 256, rngs); torch.cuda.synchronize(); t.append(time.perf_counter())
res = T.lloyd_iterate_batched(Pd, init, tc); torch.cuda.synchronize(); t.append(time.perf_counter())
names = ["sample", "to f64", "validate", "stack+check", "upload", "k-means++", "Lloyd"]
print(" ".join(f"{n}={1e3 * (b - a):.0f}ms" for n, a, b in zip(names, t[:-1], t[1:])), f"total={1e3 * (t[-1] - t[0]):.0f}ms")
