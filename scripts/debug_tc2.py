"""Small correctness run of the tensor-core encode (CSPQ_TC_KERNEL selects v1/v2) against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from oracle import oracle as O
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
for (n, m, sub, u8) in [(128, 1, 8, False), (1000, 3, 8, False), (5000, 16, 8, False), (3000, 32, 4, True), (20000, 96, 8, False)]:
    if u8:
        X = rng.integers(0, 256, (n, m * sub), dtype=np.uint8); rm = (rng.uniform(0, 255, (m, 256, sub))).astype(np.float32)
    else:
        X = rng.standard_normal((n, m * sub)).astype(np.float32); rm = (rng.standard_normal((m, 256, sub)) * 0.5).astype(np.float32)
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
    want = O.encode(X, cs.rowmajor, cs.biases, O.VARIANT_REFORM)
    got = P.encode_dataset_device(torch.from_numpy(X).to(dev), cs, P.ExecutionPlan(mode="tensor")).cpu().numpy()
    bad = np.argwhere(got != want)
    print(n, m, sub, u8, "mismatches", len(bad), bad[:5].tolist(), [(int(got[i, j]), int(want[i, j])) for i, j in bad[:5]], flush=True)
