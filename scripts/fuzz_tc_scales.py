"""Fuzz of the tensor-core encode across magnitudes (fp16 operand scaling): codebooks and rows at
random powers of two from 2^-80 to 2^70, per-coordinate and per-centroid spreads, rows far
larger / smaller than their codebook, uint8 rows.  Every code must equal the oracle's.
argv: trials [seed]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from oracle import oracle as O
trials = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(seed)
bad = 0
for t in range(trials):
    sub = int(rng.choice([4, 8])); m = int(rng.integers(1, 9)); n = int(rng.integers(1, 6000))
    u8 = rng.random() < 0.25
    rm = rng.standard_normal((m, 256, sub))
    ce = rng.integers(-80, 70, m)                         # codebook scale per subspace
    rm *= np.exp2(ce)[:, None, None]
    if rng.random() < 0.5: rm *= np.exp2(rng.integers(-14, 1, (m, 1, sub)))      # coordinate spread
    if rng.random() < 0.5: rm *= np.exp2(rng.integers(-16, 1, (m, 256, 1)))      # centroid spread
    if rng.random() < 0.3: rm[:, rng.integers(0, 256)] = 0.0
    rm = rm.astype(np.float32)
    if u8:
        X = rng.integers(0, 256, (n, m * sub), dtype=np.uint8)
        Xf = X.astype(np.float32)
    else:
        Xv = rng.standard_normal((n, m, sub)) * np.exp2(ce)[None, :, None]
        Xv *= np.exp2(rng.integers(-30, 31, (n, m, 1)) * (rng.random((n, m, 1)) < 0.3))   # rows off the codebook's scale
        if rng.random() < 0.5: Xv *= np.exp2(rng.integers(-14, 1, (1, m, sub)))
        with np.errstate(over="ignore"):
            X = Xv.reshape(n, m * sub).astype(np.float32)
        Xf = X
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
    want = O.encode(Xf, cs.rowmajor, cs.biases, O.VARIANT_REFORM)
    got = P.encode_dataset_device(torch.from_numpy(X).cuda(), cs, P.ExecutionPlan(mode="tensor")).cpu().numpy()
    nb = int((got != want).sum())
    if nb:
        bad += nb
        r, j = np.argwhere(got != want)[0]
        print(f"trial {t}: {nb} mismatches (sub {sub}, m {m}, n {n}, u8 {u8}); first row {r} subspace {j} scale 2^{ce[j]} got {got[r, j]} want {want[r, j]}")
print("trials", trials, "mismatching codes", bad)
sys.exit(1 if bad else 0)
