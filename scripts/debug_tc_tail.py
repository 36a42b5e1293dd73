import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from oracle import oracle as O
n, sub, m = 128, 4, 5
rng = np.random.default_rng(n * 31 + sub)
X = rng.standard_normal((n, m * sub)).astype(np.float32)
rm = rng.standard_normal((m, 256, sub)).astype(np.float32)
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
want, wbest = O.encode(X, cs.rowmajor, cs.biases, O.VARIANT_REFORM, want_best=True)
Xd = torch.from_numpy(X).cuda()
b = torch.empty((n, m), dtype=torch.float32, device="cuda")
for rep in range(3):
    got = P.encode_dataset_device(Xd, cs, P.ExecutionPlan(mode="tensor"), best=b).cpu().numpy()
    bb = b.cpu().numpy()
    bad = np.argwhere(got != want)
    print("rep", rep, "mismatches", len(bad))
    for i, j in bad[:10]:
        x = X[i, j*sub:(j+1)*sub].astype(np.float64)
        s = cs.biases[j].astype(np.float64) - rm[j].astype(np.float64) @ x
        o = np.argsort(s)
        print(f"  row {i} sub {j}: got {got[i,j]} want {want[i,j]} tc_best {bb[i,j]:.7g} oracle_best {wbest[i,j]:.7g} "
              f"top3 {o[:3]} {s[o[:3]]} s[got]={s[got[i,j]]:.7g}")
