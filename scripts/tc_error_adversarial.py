"""Adversarial search for the tensor-core score error |S_tc - s_oracle| / W on winners
(W = max|b| + ||x|| max||c||, per (row, subspace)).  Families: mixed-sign cancellation
inside each K = 8 group, products of widely different exponents, tf32 hi/lo split extremes
(lo parts maximal / zero / at the rounding boundary), bias >> x.c and bias << x.c; then a
hill-climb that mutates the worst pairs.  Prints max err/W per family vs the guard constant E."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_25521_b200 as P
from oracle import oracle as O

E = {8: (4 / 2**22 + 4 / 2**22 * (1 + 1 / 1024) + 9 / 2**24) * 1.01,
     4: (4 / 2**22 + 2 / 2**22 * (1 + 1 / 1024) + 5 / 2**24) * 1.01}


def err_over_w(X, rm):
    """-> per-(row, subspace) err/W on rows whose tensor code equals the oracle's (others 0)."""
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(rm.shape[0])])
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    b = torch.empty((X.shape[0], cs.m), dtype=torch.float32, device="cuda")
    codes = P.encode_dataset_device(Xd, cs, P.ExecutionPlan(mode="tensor"), best=b).cpu().numpy()
    want, wbest = O.encode(X, cs.rowmajor, cs.biases, O.VARIANT_REFORM, want_best=True, threads=os.cpu_count())
    sub = cs.sub_dim
    xs = X.astype(np.float64).reshape(X.shape[0], cs.m, sub)
    nrm = np.sqrt((xs ** 2).sum(-1))
    bmax = np.abs(cs.biases.astype(np.float64)).max(axis=1)
    cmax = np.sqrt((cs.rowmajor.astype(np.float64) ** 2).sum(-1)).max(axis=1)
    W = bmax[None, :] + nrm * cmax[None, :]
    err = np.abs(b.cpu().numpy().astype(np.float64) - wbest.astype(np.float64))
    r = np.where((codes == want) & (W > 0) & np.isfinite(err), err / np.where(W > 0, W, 1), 0.0)
    return r


def copies(rng, pat, m, jitter):
    """(m, 256, sub) codebooks: 256 jittered copies of one pattern per subspace (keeps W tight)."""
    c = np.repeat(pat[:, None, :], 256, axis=1)
    return (c * (1 + jitter * rng.standard_normal(c.shape))).astype(np.float32)


def families(rng, sub, n=20000, m=8):
    signs = lambda *s: rng.choice([-1.0, 1.0], s)
    out = {}
    # 1 mixed-sign cancellation: x_t c_t = +-A alternating inside each group of 8 products
    A = 10.0 ** rng.uniform(-2, 3, (m, 1))
    cpat = A * signs(m, sub)
    alt = np.tile([1.0, -1.0], sub // 2)
    X = (np.abs(A.T)[:, :, None] * alt[None, None, :] * np.sign(cpat)[None, :, :]
         * (1 + 1e-3 * rng.standard_normal((n, m, sub))))
    out["cancel"] = (X.reshape(n, m * sub), copies(rng, cpat, m, 1e-3))
    # 2 exponent spread inside a group: products from 2^-30 to 2^30
    e = rng.integers(-15, 16, (n, m, sub))
    X = signs(n, m, sub) * 2.0 ** e * (1 + rng.random((n, m, sub)))
    cpat = signs(m, sub) * 2.0 ** rng.integers(-15, 16, (m, sub)) * (1 + rng.random((m, sub)))
    out["exp_spread"] = (X.reshape(n, m * sub), copies(rng, cpat, m, 1e-4))
    # 3 tf32 split extremes: lo part maximal (just under half a tf32 ulp), zero, at the tie
    base = 1.0 + rng.integers(0, 1024, (n, m, sub)) / 1024.0
    lo = rng.choice([0.0, 0.4999, 0.5, -0.4999, 0.25], (n, m, sub)) / 1024.0
    X = signs(n, m, sub) * base * (1 + lo) * 2.0 ** rng.integers(-4, 5, (n, m, sub))
    cb = 1.0 + rng.integers(0, 1024, (m, sub)) / 1024.0
    cpat = signs(m, sub) * cb * (1 + 0.4999 / 1024) * 2.0 ** rng.integers(-4, 5, (m, sub))
    out["tf32_split"] = (X.reshape(n, m * sub), copies(rng, cpat, m, 1e-5))
    # 4 bias >> x.c: far-off centroids, small x
    cpat = 1000.0 + rng.standard_normal((m, sub))
    X = 1e-2 * rng.standard_normal((n, m * sub))
    out["bias_dominant"] = (X, copies(rng, cpat, m, 1e-3))
    # 5 bias << x.c: small centroids, huge x
    cpat = 1e-2 * rng.standard_normal((m, sub))
    X = 1e4 * rng.standard_normal((n, m * sub))
    out["dot_dominant"] = (X, copies(rng, cpat, m, 1e-1))
    # 6 x ~ c (winner near the row itself): scores near -|c|^2/2, cancellation b - x.c
    cpat = rng.standard_normal((m, sub)) * 10
    X = np.repeat(cpat.reshape(1, m * sub), n, 0) * (1 + 1e-6 * rng.standard_normal((n, m * sub)))
    out["self_cancel"] = (X, copies(rng, cpat, m, 1e-6))
    return {k: (np.ascontiguousarray(x, dtype=np.float32), np.ascontiguousarray(c, dtype=np.float32))
            for k, (x, c) in out.items()}


def climb(rng, X, rm, rounds=int(os.environ.get("TC_CLIMB_ROUNDS", "4")), keep=256):
    """Mutate the worst rows (fresh jitter of their values, same codebooks)."""
    sub = rm.shape[2]
    worst = 0.0
    for _ in range(rounds):
        r = err_over_w(X, rm)
        worst = max(worst, float(r.max()))
        top = np.argsort(r.max(axis=1))[-keep:]
        seeds = X[top]
        reps = max(1, X.shape[0] // keep)
        Xn = np.repeat(seeds, reps, 0)
        scale = 10.0 ** rng.uniform(-7, -2, (Xn.shape[0], 1))
        Xn = Xn * (1 + scale * rng.standard_normal(Xn.shape))
        X = np.ascontiguousarray(Xn, dtype=np.float32)
    return worst


def main():
    rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
    res = {}
    for sub in (8, 4):
        for name, (X, rm) in families(rng, sub).items():
            w = climb(rng, X, rm)
            res[(sub, name)] = w
            print(f"sub {sub} {name:14s} max err/W {w:.3e}  = {w / E[sub]:.3f} E  (E = {E[sub]:.3e})", flush=True)
    return res


if __name__ == "__main__":
    main()
