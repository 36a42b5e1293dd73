"""Layout fuzz of the tcgen05 encode: random n, m, d_sub, input dtype, row strides wider than d (views into a
wider matrix, 16-byte aligned offsets), strided `out` rows -- tensor mode against the independent exact SIMT
kernel.  Run on a GPU box: python scripts/fuzz_tc_layouts.py [cases] [seed]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
dev = torch.device("cuda", 0)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for c in range(cases):
    sub = int(rng.choice([4, 8])); m = int(rng.integers(1, 41)); d = m * sub
    n = int(rng.choice([1, 2, 31, 127, 128, 129, 255, 1000, 1025, 4097, int(rng.integers(1, 20000))]))
    u8 = bool(rng.integers(0, 2))
    align = 16 if not u8 else sub                       # elements: float rows need 16-byte alignment, byte rows d_sub
    step = (4 if not u8 else sub)
    pad_l = int(rng.integers(0, 4)) * step; pad_r = int(rng.integers(0, 4)) * step
    wide = d + pad_l + pad_r
    if u8:
        W = torch.from_numpy(rng.integers(0, 256, (n, wide), dtype=np.uint8)).to(dev)
    else:
        W = torch.from_numpy((rng.standard_normal((n, wide)) * float(rng.choice([1e-3, 1.0, 50.0]))).astype(np.float32)).to(dev)
    X = W[:, pad_l:pad_l + d]
    rows = X[torch.from_numpy(rng.integers(0, n, 256)).to(dev)].float().cpu().numpy()
    rows = rows + rng.standard_normal(rows.shape).astype(np.float32) * (0.01 * (np.abs(rows).max() + 1e-3))
    rm = np.ascontiguousarray(rows.reshape(256, m, sub).transpose(1, 0, 2))
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
    outw = torch.full((n, m + int(rng.integers(0, 3)) * 16), 255, dtype=torch.uint8, device=dev)
    out = outw[:, :m]
    got = P.encode_dataset_device(X, cs, P.ExecutionPlan(mode="tensor"), out=out)
    want = P.encode_dataset_device(X.contiguous(), cs, P.ExecutionPlan(mode="exact"))
    ok = torch.equal(got, want) and bool((outw[:, m:] == 255).all())
    if not ok:
        bad += 1
        print(f"case {c}: MISMATCH n={n} m={m} sub={sub} u8={u8} pad=({pad_l},{pad_r}) out_w={outw.shape[1]} diff={(got != want).sum().item()}")
print(f"{cases} cases, {bad} bad")
sys.exit(1 if bad else 0)
