"""Parity of the GPU Lloyd / k-means++ path with the reference's golden runs
and the oracle, mirroring pkg/tests/test_training.py."""

import numpy as np
import pytest

from conftest import cases, golden, group

pytestmark = pytest.mark.gpu

LLOYD = golden("lloyd_golden.npz")
TRAIN = golden("train_golden.npz")


@pytest.fixture(scope="module")
def P():
    import paper_2605_25521_b200 as P
    return P


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return (np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)).max()


@pytest.mark.parametrize("case", cases(LLOYD))
def test_lloyd_vs_reference_golden(P, case):
    g = group(LLOYD, case)
    cfg = P.TrainConfig(k=g["init"].shape[0], max_iters=int(g["max_iters"]), tol=float(g["tol"]))
    r = P.lloyd_iterate(g["pts"].astype(np.float64), g["init"], cfg)
    assert r.iterations == int(g["iterations"])
    assert np.array_equal(r.assignments, g["assignments"])
    assert rel_err(r.centroids, g["centroids"]) <= 1e-5
    np.testing.assert_allclose(r.objectives, g["objectives"], rtol=1e-12, atol=1e-12)
    # float64 norms in np.einsum's order: in fact bit for bit
    assert r.centroids.tobytes() == g["centroids"].tobytes()
    assert np.asarray(r.objectives).tobytes() == g["objectives"].tobytes()


@pytest.mark.parametrize("case", cases(LLOYD))
def test_lloyd_vs_oracle_bitwise(P, oracle, case):
    g = group(LLOYD, case)
    pts = g["pts"].astype(np.float64)
    o = oracle.lloyd(pts, g["init"], int(g["max_iters"]), float(g["tol"]))
    r = P.lloyd_iterate(pts, g["init"], P.TrainConfig(k=g["init"].shape[0], max_iters=int(g["max_iters"]),
                                                      tol=float(g["tol"])))
    assert r.iterations == o["iterations"]
    assert r.centroids.tobytes() == o["centroids"].tobytes()
    assert np.array_equal(r.assignments, o["assignments"])
    assert r.objectives == o["objectives"]


def test_batched_subspaces_stop_independently(P, oracle):
    rng = np.random.default_rng(5)
    m, n, sub, k = 6, 3000, 4, 32
    pts = []
    for j in range(m):
        cen = rng.uniform(-5, 5, (k, sub)) * (j + 1)
        pts.append((cen[rng.integers(0, k, n)] + rng.normal(0, 0.3 + 0.2 * j, (n, sub))).astype(np.float32))
    init = np.stack([p[np.sort(rng.choice(n, k, replace=False))] for p in pts]).astype(np.float64)
    cfg = P.TrainConfig(k=k, max_iters=30, tol=1e-3)
    res = P.lloyd_iterate_batched(np.stack(pts), init, cfg)
    iters = set()
    for j in range(m):
        o = oracle.lloyd(pts[j].astype(np.float64), init[j], 30, 1e-3)
        assert res[j].iterations == o["iterations"]
        assert res[j].centroids.tobytes() == o["centroids"].tobytes()
        assert res[j].objectives == o["objectives"]
        iters.add(res[j].iterations)
    assert len(iters) > 1  # subspaces really stopped at different iterations


def test_kmeanspp_default_path_vs_reference(P):
    """train_all_codebooks_report with the reference's defaults (per-subspace
    sampling + k-means++ + tol stop) against the reference's own run."""
    X = TRAIN["kmpp/X"]
    params = P.PQParams(d=32, m=4, k=64)
    cfg = P.TrainConfig(k=64, seed=11, sample_cap=3000, max_iters=12)
    cbs, reps = P.train_all_codebooks_report(P.VectorDataset(data=np.array(X)), params, cfg)
    ref = TRAIN["kmpp/centroids"]
    for j in range(4):
        assert reps[j].iterations == int(TRAIN[f"kmpp/iterations_{j}"])
        assert np.array_equal(reps[j].assignments, TRAIN[f"kmpp/assignments_{j}"])
        assert rel_err(cbs[j].centroids_rowmajor, ref[j]) <= 1e-5
        np.testing.assert_allclose(reps[j].objectives, TRAIN[f"kmpp/objectives_{j}"], rtol=1e-12)
        assert cbs[j].biases.tobytes() == P.compute_biases(cbs[j].centroids_rowmajor).tobytes()


def test_kmeanspp_seeding_matches_reference(P):
    from paper_2605_25521_b200.training import _sample, _subspace_rngs, kmeanspp_init_batched
    X = TRAIN["kmpp/X"]
    rngs = _subspace_rngs(11, 4)
    pts = np.ascontiguousarray(X[:, 8:16])
    sampled = _sample(pts, 3000, rngs[1])
    init = kmeanspp_init_batched([sampled.astype(np.float64)], 64, [rngs[1]])[0]
    assert init.tobytes() == TRAIN["kmpp/seed_init_sub1"].tobytes()


# ---- pkg/tests/test_training.py on the GPU ----

def test_separable_pair(P):
    cb, rep = P.train_codebook_report(np.array([[0.0], [10.0]], np.float32), P.TrainConfig(k=2, seed=0))
    assert sorted(cb.centroids_rowmajor[:, 0].tolist()) == [0.0, 10.0]
    assert rep.objectives[-1] == 0.0


def test_single_cluster_mean(P):
    cb, rep = P.train_codebook_report(np.array([[1.0], [3.0]], np.float32), P.TrainConfig(k=1, seed=0))
    assert cb.centroids_rowmajor[0, 0] == pytest.approx(2.0)
    assert rep.objectives[-1] == pytest.approx(2.0)


def test_training_errors(P):
    with pytest.raises(P.TrainingError):
        P.train_codebook(np.zeros((2, 3), np.float32), P.TrainConfig(k=5))
    with pytest.raises(P.TrainingError, match="degenerate"):
        P.train_codebook(np.full((50, 2), 7.0, np.float32), P.TrainConfig(k=2))
    data = np.array([[0.0, 5.0], [10.0, 5.0]], np.float32)
    with pytest.raises(P.TrainingError, match="subspace 1"):
        P.train_all_codebooks(data, P.PQParams(d=2, m=2, k=2), P.TrainConfig(k=2, seed=0))


def test_k1_means_raw_array(P):
    data = np.array([[0.0, 5.0], [10.0, 5.0]], np.float32)
    cbs = P.train_all_codebooks(data, P.PQParams(d=2, m=2, k=1), P.TrainConfig(k=1, seed=0))
    assert cbs[0].centroids_rowmajor[0, 0] == pytest.approx(5.0)
    assert cbs[1].centroids_rowmajor[0, 0] == pytest.approx(5.0)


def _synth(n, d, clusters, seed, noise=0.05):
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.uniform(-1.0, 1.0, size=(clusters, d)).astype(np.float32)
    labels = rng.integers(0, clusters, size=n)
    return (means[labels] + rng.normal(0.0, noise, size=(n, d)).astype(np.float32)).astype(np.float32)


def test_monotone_deterministic_consistent(P):
    X = _synth(4000, 16, 8, 0)
    params, cfg = P.PQParams(d=16, m=2, k=32), P.TrainConfig(k=32, seed=0)
    a, reps = P.train_all_codebooks_report(X, params, cfg)
    for rep in reps:
        for x, y in zip(rep.objectives, rep.objectives[1:]):
            assert y <= x * (1 + 1e-4)
    b = P.train_all_codebooks(X, params, cfg)
    for x, y in zip(a, b):
        assert x.centroids_rowmajor.tobytes() == y.centroids_rowmajor.tobytes()
    pts = X[:1500, :8]
    cb, rep = P.train_codebook_report(pts, P.TrainConfig(k=16, seed=5))
    for i in range(0, 1500, 97):
        assert P.encode_ref(pts[i], cb) == rep.assignments[i]


def test_sample_cap_and_repair(P):
    pts = _synth(5000, 4, 4, 6)
    _, rep = P.train_codebook_report(pts, P.TrainConfig(k=4, seed=6, sample_cap=500))
    assert rep.n_train == 500
    _, rep = P.train_codebook_report(pts, P.TrainConfig(k=4, seed=6, sample_cap=0))
    assert rep.n_train == 5000
    res = P.lloyd_iterate(np.array([[0.0], [0.1], [0.2], [10.0], [10.1], [50.0]]),
                          np.array([[0.0], [0.0], [10.0]]), P.TrainConfig(k=3, max_iters=10, seed=0))
    assert np.all(np.bincount(res.assignments, minlength=3) >= 1)
    assert any(abs(c - 50.0) < 1e-6 for c in res.centroids[:, 0])


def test_subspace_independence(P):
    X = _synth(2000, 8, 4, 3)
    cfg = P.TrainConfig(k=8, seed=77)
    cbs = P.train_all_codebooks(X, P.PQParams(d=8, m=2, k=8), cfg)
    solo = P.train_codebook(X[:, 4:8], cfg, subspace_index=1)
    assert cbs[1].centroids_rowmajor.tobytes() == solo.centroids_rowmajor.tobytes()


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_config_training_vs_oracle(P, oracle, name):
    """Config-shaped training (sample-point init, tol 0) at reduced sample
    size: GPU == oracle bit for bit for a few subspaces."""
    import torch
    from paper_2605_25521_b200 import configs as C
    cfg = C.CONFIGS[name].scaled(n=200_000, n_train=20_000)
    dev = torch.device("cuda", 0)
    S = C.training_sample(cfg, dev)
    Ssm = C.subspace_major(S, cfg.m)[:4]
    init = C.lloyd_init(cfg, Ssm)
    res = P.lloyd_iterate_batched(Ssm, init, P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0))
    Sh = Ssm.cpu().numpy()
    for j in range(4):
        o = oracle.lloyd(Sh[j].astype(np.float64), init[j], cfg.iters, 0.0)
        assert res[j].iterations == o["iterations"]
        assert res[j].centroids.tobytes() == o["centroids"].tobytes(), (name, j)
        assert res[j].objectives == o["objectives"]


def test_sharded_driver_matches_batched_lloyd(P):
    """distributed.lloyd_sharded on the CUDA step backend (world size 1, both
    reduce modes) reproduces cspq_lloyd_train bit for bit."""
    import torch
    from paper_2605_25521_b200.distributed import CudaSteps, lloyd_sharded
    rng = np.random.default_rng(12)
    m, n, sub, k = 3, 4000, 8, 64
    pts = rng.standard_normal((m, n, sub)).astype(np.float32)
    init = pts[:, :k].astype(np.float64).copy()
    init[:, 5] = init[:, 4]
    cfg = P.TrainConfig(k=k, max_iters=12, tol=1e-5)
    ref = P.lloyd_iterate_batched(pts, init, cfg)
    dev = torch.device("cuda", 0)
    Pd = torch.from_numpy(pts).to(dev)
    for mode in ("allgather", "allreduce"):
        res = lloyd_sharded(CudaSteps(Pd, 0, n, m, sub, k, dev), torch.from_numpy(init).to(dev), cfg, reduce=mode)
        for a, b in zip(res, ref):
            assert a.iterations == b.iterations
            assert a.centroids.tobytes() == b.centroids.tobytes()
            assert a.objectives == b.objectives
            assert np.array_equal(a.assignments, b.assignments)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_tensor_screened_assignment_equals_float64(P, monkeypatch, name):
    """k = 256, sub in {4, 8}: the assignment runs through the tcgen05 encode
    kernel (mark mode) plus a float64 settle of flagged points.  Every
    subspace's centroids, objectives, iterations and final assignments equal
    the plain float64 kernel's (CSPQ_LLOYD_TC=0) bit for bit."""
    import torch
    from paper_2605_25521_b200 import configs as C
    cfg = C.CONFIGS[name].scaled(n=200_000, n_train=50_000)
    S = C.training_sample(cfg, torch.device("cuda", 0))
    Ssm = C.subspace_major(S, cfg.m)
    init = C.lloyd_init(cfg, Ssm)
    tc = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
    monkeypatch.setenv("CSPQ_LLOYD_TC", "0")
    ref = P.lloyd_iterate_batched(Ssm, init, tc)
    monkeypatch.setenv("CSPQ_LLOYD_TC", "1")
    got = P.lloyd_iterate_batched(Ssm, init, tc)
    for j in range(cfg.m):
        assert got[j].centroids.tobytes() == ref[j].centroids.tobytes(), (name, j)
        assert got[j].objectives == ref[j].objectives and got[j].iterations == ref[j].iterations
        assert np.array_equal(got[j].assignments, ref[j].assignments)


def test_tensor_screened_assignment_ties(P, monkeypatch, oracle):
    """Heavy exact ties (few distinct points, duplicated initial centroids,
    empty clusters): flagged points settle in float64 with the first index."""
    rng = np.random.default_rng(5)
    m, n, sub, k = 2, 6000, 8, 256
    base = np.round(rng.uniform(-3, 3, (40, sub))).astype(np.float32)
    pts = np.ascontiguousarray(base[rng.integers(0, 40, (m, n))])
    init = np.ascontiguousarray(pts[:, rng.integers(0, n, k)].astype(np.float64))
    tc = P.TrainConfig(k=k, max_iters=6, tol=0.0)
    monkeypatch.setenv("CSPQ_LLOYD_TC", "1")
    got = P.lloyd_iterate_batched(pts, init, tc)
    for j in range(m):
        o = oracle.lloyd(pts[j].astype(np.float64), init[j], 6, 0.0)
        assert got[j].centroids.tobytes() == o["centroids"].tobytes()
        assert got[j].objectives == o["objectives"]
        assert np.array_equal(got[j].assignments, o["assignments"])


@pytest.mark.parametrize("sub", [4, 8])
def test_screened_final_pass_far_from_origin(P, monkeypatch, oracle, sub):
    """The final float32 REFERENCE pass (training.py:143-150) is screened by
    the tensor kernel with a band widened for the REFERENCE's own rounding:
    points far from the origin make |x|^2 dominate (vv + cc_l) - 2 dd_l, so
    the REFERENCE rounds many real gaps away (exact ties and swapped orders);
    every such point must be flagged and rescanned.  Final assignments and
    objectives equal the plain REFERENCE kernel's and the oracle's."""
    rng = np.random.default_rng(11 + sub)
    m, n, k = 3, 20_000, 256
    pts = (1000.0 + rng.standard_normal((m, n, sub)) * np.array([0.5, 2.0, 8.0])[:, None, None]).astype(np.float32)
    init = np.ascontiguousarray(pts[:, rng.choice(n, k, replace=False)].astype(np.float64))
    cfg = P.TrainConfig(k=k, max_iters=3, tol=0.0)
    monkeypatch.setenv("CSPQ_LLOYD_TC", "0")
    ref = P.lloyd_iterate_batched(pts, init, cfg)
    monkeypatch.setenv("CSPQ_LLOYD_TC", "1")
    got = P.lloyd_iterate_batched(pts, init, cfg)
    for j in range(m):
        assert np.array_equal(got[j].assignments, ref[j].assignments), j
        assert got[j].objectives == ref[j].objectives
        o = oracle.lloyd(pts[j].astype(np.float64), init[j], 3, 0.0)
        assert np.array_equal(got[j].assignments, o["assignments"]), j
        assert got[j].objectives == o["objectives"]


def test_screened_assignment_on_row_ranges(P, monkeypatch):
    """cspq_lloyd_assign over disjoint point ranges [b, e) (the row-sharded
    driver's call) equals one full-range call and the plain float64 kernel."""
    import torch
    from paper_2605_25521_b200.distributed import CudaSteps
    rng = np.random.default_rng(21)
    m, n, sub, k = 3, 10_001, 8, 256
    dev = torch.device("cuda", 0)
    pts = torch.from_numpy(rng.standard_normal((m, n, sub)).astype(np.float32)).to(dev)
    C64 = torch.from_numpy(rng.standard_normal((m, k, sub))).to(dev)
    state = torch.ones(m, dtype=torch.int32, device=dev)
    steps = CudaSteps(pts, 0, n, m, sub, k, dev)

    def run(ranges, tc):
        monkeypatch.setenv("CSPQ_LLOYD_TC", tc)
        a = torch.full((m, n), -1, dtype=torch.int32, device=dev)
        s = torch.full((m, n), -1.0, dtype=torch.float64, device=dev)
        for b, e in ranges:
            steps.assign(C64, state, b, e, a, s)
        torch.cuda.synchronize()
        return a.cpu().numpy(), s.cpu().numpy()

    full = run([(0, n)], "0")
    for ranges in ([(0, n)], [(0, 3000), (3000, 7777), (7777, n)], [(5, 133), (0, 5), (133, n)]):
        got = run(ranges, "1")
        assert np.array_equal(got[0], full[0]) and got[1].tobytes() == full[1].tobytes(), ranges


KPPZ = golden("kpp_zero_golden.npz")


@pytest.mark.parametrize("case", cases(KPPZ))
def test_kmeanspp_zero_mass_switches_to_integer_draws(P, case):
    """training.py:84-86: once the D^2 mass is zero the reference draws rng.integers(n) for
    the remaining seeds; the GPU seeding reports the step and the host replays the draws --
    same seeds, and the generator ends in the reference's state."""
    from paper_2605_25521_b200.training import kmeanspp_init_batched
    g = group(KPPZ, case)
    rng = np.random.default_rng(int(g["seed"]))
    init = kmeanspp_init_batched([g["pts"].astype(np.float64)], int(g["k"]), [rng])[0]
    assert init.tobytes() == g["init"].tobytes()
    assert int(rng.integers(1 << 30)) == int(g["next_draw"])
