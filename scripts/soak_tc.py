"""Soak of the tcgen05 encode: many launches of random shapes (n up to 300K rows, m up to 192, d_sub 4 / 8, f32 / u8
rows, fix-up and mark-mode through a short Lloyd run now and then); every launch must return (a lost mbarrier arrival
traps after ~10 s) and every 10th is compared with the exact SIMT kernel.  python scripts/soak_tc.py [seconds] [seed]."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
dev = torch.device("cuda", 0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0 = time.time(); launches = checked = bad = 0
while time.time() - t0 < budget:
    sub = int(rng.choice([4, 8])); m = int(rng.choice([1, 2, 3, 5, 16, 32, 96, 120, 192])); d = m * sub
    u8 = bool(rng.integers(0, 2))
    n = int(rng.choice([1, 127, 129, 4096, 4097, int(rng.integers(1, 300000))]))
    if n * d > 60_000_000: n = 60_000_000 // d
    X = (torch.randint(0, 256, (n, d), dtype=torch.uint8, device=dev) if u8
         else torch.randn((n, d), device=dev) * float(rng.choice([0.03, 1.0, 20.0])))
    rows = X[torch.randint(0, n, (256,), device=dev)].float().cpu().numpy()
    rows = rows + rng.standard_normal(rows.shape).astype(np.float32) * (0.02 * (np.abs(rows).max() + 1e-3))
    rm = np.ascontiguousarray(rows.reshape(256, m, sub).transpose(1, 0, 2))
    cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
    reps = int(rng.integers(1, 6))
    for _ in range(reps):
        got = P.encode_dataset_device(X, cs, P.ExecutionPlan(mode="tensor"))
        launches += 1
    torch.cuda.synchronize()
    if launches % 10 < reps:
        want = P.encode_dataset_device(X, cs, P.ExecutionPlan(mode="exact"))
        checked += 1
        if not torch.equal(got, want):
            bad += 1
            print(f"MISMATCH n={n} m={m} sub={sub} u8={u8}: {(got != want).sum().item()} codes", flush=True)
    if not u8 and n >= 2048 and rng.integers(0, 8) == 0:  # mark mode: a 3-iteration Lloyd run, twice, identical
        S = X[:min(n, 20000)].reshape(-1, m, sub).permute(1, 0, 2).contiguous()
        init = S[:, :256].double().cpu().numpy() if S.shape[1] >= 256 else None
        if init is not None and np.unique(init.reshape(m, 256, -1)[0], axis=0).shape[0] == 256:
            tc = P.TrainConfig(k=256, max_iters=3, tol=0.0)
            a = P.lloyd_iterate_batched(S, init, tc, return_assignments=False)
            b = P.lloyd_iterate_batched(S, init, tc, return_assignments=False)
            if any(not np.array_equal(x.centroids, y.centroids) for x, y in zip(a, b)):
                bad += 1
                print("Lloyd runs differ", flush=True)
print(f"{launches} launches, {checked} checked against the exact kernel, {bad} bad, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
