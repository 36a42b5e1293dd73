"""encode_dataset on a pageable numpy array (the reference's usual call): page-locking the
caller's array for the call (cudaHostRegister, CSPQ_HOST_REGISTER=1) vs staging each batch
through the pinned ring (CSPQ_HOST_REGISTER=0), and pinned host buffers for comparison."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
cfg = C.CONFIGS["c3"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
Xd = C.generate(cfg, 0, n, torch.device("cuda", 0))
X = Xd.cpu().numpy().copy()                      # pageable
rng = np.random.default_rng(0)
rm = (rng.standard_normal((cfg.m, 256, cfg.sub)) * 0.2).astype(np.float32)
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
want = P.encode_dataset_device(Xd, cs).cpu().numpy()
P.encode_dataset(X[:100000], cs)
pinned = P.pinned_empty(X.shape, np.float32)
pinned[:] = X
for label, arr, reg in (("staged", X, "0"), ("register", X, "1"), ("pinned", pinned, "0"),
                        ("staged", X, "0"), ("register", X, "1"), ("pinned", pinned, "0")):
    os.environ["CSPQ_HOST_REGISTER"] = reg
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    codes = P.encode_dataset(arr, cs).codes
    dt = time.perf_counter() - t0
    assert np.array_equal(codes, want)
    print(f"{label:9s} n={n}: {n / dt / 1e6:6.2f} M vec/s ({n * cfg.d * 4 / dt / 1e9:5.1f} GB/s of rows)", flush=True)
