"""Parity of the CUDA encode path with the oracle and the reference's golden
vectors (bit-exact codes and scores), mirroring the reference's own hot-path
tests (pkg/tests/test_kernels.py, test_bulk.py, test_acceptance.py 1-4)."""

import numpy as np
import pytest

from conftest import cases, golden, group

pytestmark = pytest.mark.gpu

ENC = golden("encode_golden.npz")
MODES = ("auto", "exact", "guarded")


@pytest.fixture(scope="module")
def P():
    import paper_2605_25521_b200 as P
    import torch
    assert torch.cuda.is_available()
    return P


def cset_of(P, rowmajor, biases=None):
    rm = np.ascontiguousarray(rowmajor, dtype=np.float32)
    cbs = [P.Codebook.from_rowmajor(j, rm[j]) for j in range(rm.shape[0])]
    cs = P.CodebookSet.from_codebooks(cbs)
    if biases is not None:
        assert cs.biases.tobytes() == np.asarray(biases, np.float32).tobytes()
    return cs


def device_codes(P, X, cs, variant, mode="auto", precomputed_bias=True):
    import torch
    Xd = torch.from_numpy(np.array(X, copy=True, order="C")).cuda()
    plan = P.ExecutionPlan(variant=variant, mode=mode)
    out = P.encode_dataset_device(Xd, cs, plan, precomputed_bias=precomputed_bias)
    torch.cuda.synchronize()
    c = out.cpu().numpy()
    return c.view(np.uint16) if c.dtype == np.int16 else c


@pytest.mark.parametrize("case", cases(ENC))
@pytest.mark.parametrize("mode", MODES)
def test_golden_codes_device(P, case, mode):
    g = group(ENC, case)
    cs = cset_of(P, g["rowmajor"], g["biases"])
    EV = P.EncoderVariant
    for var, key in ((EV.REFERENCE, "codes_reference"), (EV.REFORMULATED, "codes_reformulated"),
                     (EV.BLOCKED, "codes_blocked")):
        got = device_codes(P, g["X"], cs, var, mode)
        assert got.tobytes() == g[key].tobytes(), (case, key, mode, int((got != g[key]).sum()))
    got = device_codes(P, g["X"], cs, EV.BLOCKED, mode, precomputed_bias=False)
    assert got.tobytes() == g["codes_nobias"].tobytes()


@pytest.mark.parametrize("case", cases(ENC))
def test_golden_codes_host_pipeline(P, case):
    g = group(ENC, case)
    cs = cset_of(P, g["rowmajor"])
    for batch in (1, 7, 4096):
        plan = P.ExecutionPlan(batch_rows=batch, streams=3)
        got = P.encode_dataset(g["X"], cs, plan).codes
        assert got.tobytes() == g["codes_blocked"].tobytes(), (case, batch)


@pytest.mark.parametrize("case", [c for c in cases(ENC) if not c.startswith("nonfinite")])
def test_golden_scores_bitwise(P, case):
    g = group(ENC, case)
    cs = cset_of(P, g["rowmajor"])
    nb = g["best_reformulated"].shape[0]
    sub = cs.sub_dim
    for i in range(min(nb, 6)):
        for j in range(cs.m):
            v = np.asarray(g["X"][i, j * sub:(j + 1) * sub], np.float32)
            code, s = P.encode_reform_with_score(v, cs[j])
            assert s.tobytes() == g["best_reformulated"][i, j].tobytes()
            assert code == g["codes_reformulated"][i, j]
            code, s = P.encode_ref_with_score(v, cs[j])
            assert s.tobytes() == g["best_reference"][i, j].tobytes()
            code, s = P.encode_blocked_with_score(v, cs[j], w=4)
            assert s.tobytes() == g["best_reformulated"][i, j].tobytes()


# ---- the reference's kernel tests (pkg/tests/test_kernels.py), on the GPU ----

def cb_from(P, rows, j=0):
    return P.Codebook.from_rowmajor(j, np.asarray(rows, dtype=np.float32))


def test_known_answers(P):
    assert P.encode_ref([1, 0], cb_from(P, [[1, 0], [0, 1]])) == 0
    assert P.encode_ref([0.6, 0.4], cb_from(P, [[1, 0], [0, 1]])) == 0
    assert P.encode_ref([1, 0], cb_from(P, [[1, 0], [1, 0]])) == 0
    cb = cb_from(P, [[3, 4]])
    code, s = P.encode_reform_with_score([1, 0], cb)
    _, d = P.encode_ref_with_score([1, 0], cb)
    assert code == 0 and s == pytest.approx(9.5) and d == pytest.approx(20.0)
    cb = cb_from(P, [[1, 0], [0, 1], [2, 0], [0, 0]])
    code, s = P.encode_blocked_with_score([1, 0], cb, w=2)
    assert code == 0 and s == pytest.approx(-0.5)
    assert P.encode_reform([9.0, -3.0], cb_from(P, [[0.1, 0.2]])) == 0


def test_dim_mismatch_and_layout_errors(P):
    with pytest.raises(P.ConfigError):
        P.encode_ref([1, 0, 0], cb_from(P, [[1, 0]]))
    cb = cb_from(P, [[1.0, 2.0]])
    broken = P.Codebook(0, cb.centroids_rowmajor, cb.centroids_transposed[:, :0], cb.biases)
    with pytest.raises(P.ConfigError):
        P.encode_blocked([1.0, 2.0], broken, w=2)
    with pytest.raises(P.ConfigError):
        P.encode_blocked([1.0, 2.0], cb, w=0)


@pytest.mark.parametrize("k,w", [(8, 8), (5, 4), (3, 16), (7, 1)])
def test_blocked_equals_reform(P, k, w):
    rng = np.random.default_rng(k * 100 + w)
    rows = rng.standard_normal((k, 4)).astype(np.float32)
    cb = cb_from(P, rows)
    vs = rng.standard_normal((200, 4)).astype(np.float32)
    for v in vs:
        assert P.encode_blocked(v, cb, w=w) == P.encode_reform(v, cb)


@pytest.mark.parametrize("w", [1, 2, 4, 8, 16])
def test_duplicated_centroid_tie(P, w):
    rng = np.random.default_rng(8)
    rows = rng.standard_normal((10, 5)).astype(np.float32)
    rows[7] = rows[2]
    cb = cb_from(P, rows)
    q = rows[2]
    assert P.encode_ref(q, cb) == 2
    assert P.encode_reform(q, cb) == 2
    assert P.encode_blocked(q, cb, w=w) == 2


def test_tie_determinism_acceptance3(P):
    # test_acceptance.py:99-118 (100 crafted codebooks, every variant)
    rng = np.random.default_rng(1003)
    bad = 0
    for _ in range(100):
        rows = rng.standard_normal((32, 8)).astype(np.float32)
        i1, i2 = sorted(rng.choice(32, size=2, replace=False))
        rows[i2] = rows[i1]
        cs = P.CodebookSet.from_codebooks([cb_from(P, rows)])
        q = rows[i1][None]
        got = set()
        for var in P.EncoderVariant:
            for mode in MODES:
                got.add(int(device_codes(P, q, cs, var, mode)[0, 0]))
        bad += got != {int(i1)}
    assert bad == 0


def test_scale_invariance(P):
    rng = np.random.default_rng(9)
    rows = rng.standard_normal((25, 6)).astype(np.float32)
    cb = cb_from(P, rows)
    doubled = P.Codebook(0, np.ascontiguousarray(rows * np.float32(2)),
                         np.ascontiguousarray((rows * np.float32(2)).T), cb.biases * np.float32(2))
    for v in rng.standard_normal((100, 6)).astype(np.float32):
        assert P.encode_reform(v, cb) == P.encode_reform(v, doubled)
        assert P.encode_blocked(v, cb, w=4) == P.encode_blocked(v, doubled, w=4)


def test_encode_vector(P):
    cbs = [cb_from(P, [[1, 0], [0, 1]], 0), cb_from(P, [[1, 0], [0, 1]], 1)]
    assert P.encode_vector([1, 0, 0, 1], cbs).tolist() == [0, 1]
    rng = np.random.default_rng(10)
    cbs = [cb_from(P, rng.standard_normal((6, 3)).astype(np.float32), j) for j in range(4)]
    v = np.concatenate([cb.centroids_rowmajor[3] for cb in cbs])
    for var in P.EncoderVariant:
        assert P.encode_vector(v, cbs, var).tolist() == [3, 3, 3, 3]
    with pytest.raises(P.ConfigError):
        P.encode_vector([1, 0, 0], [cb_from(P, [[1, 0]]), cb_from(P, [[1, 0]], 1)])


# ---- bulk (pkg/tests/test_bulk.py) ----

@pytest.fixture(scope="module")
def bulk_setup(P):
    rng = np.random.default_rng(31)
    cbs = [P.Codebook.from_rowmajor(j, rng.standard_normal((24, 4)).astype(np.float32)) for j in range(3)]
    X = rng.standard_normal((1000, 12)).astype(np.float32)
    return X, cbs


def test_matches_per_vector(P, bulk_setup):
    X, cbs = bulk_setup
    small = X[:3]
    for order in (P.CHUNK_MAJOR, P.VECTOR_MAJOR):
        for var in P.EncoderVariant:
            got = P.encode_dataset(small, cbs, P.ExecutionPlan(order=order, variant=var, block_size=2)).codes
            want = np.stack([P.encode_vector(v, cbs, var) for v in small])
            assert np.array_equal(got, want)


def test_plan_invariance(P, bulk_setup):
    X, cbs = bulk_setup
    base = None
    for order in (P.CHUNK_MAJOR, P.VECTOR_MAJOR):
        for block_size in (1, 7, 64, 1000):
            for workers in (1, 3):
                for mode in MODES:
                    got = P.encode_dataset(X, cbs, P.ExecutionPlan(order=order, block_size=block_size,
                                                                    workers=workers, mode=mode,
                                                                    batch_rows=block_size)).codes
                    base = got if base is None else base
                    assert got.tobytes() == base.tobytes()


def test_multi_device_split(P, oracle):
    """ExecutionPlan(devices=...): host rows split into contiguous ranges, one pipeline per
    device from host threads (the same GPU twice / three times here: the one-GPU box still
    exercises the split, the threads and the per-range outputs); codes equal one device's
    and the oracle's, for ragged sizes, pinned and pageable input, the tensor-core and SIMT
    paths."""
    rng = np.random.default_rng(8)
    m, sub, k = 12, 8, 256
    rm = rng.standard_normal((m, k, sub)).astype(np.float32)
    cbs = [P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)]
    cs = P.CodebookSet.from_codebooks(cbs)
    for n in (1, 5, 100_003):
        X = rng.standard_normal((n, m * sub)).astype(np.float32)
        want = oracle.encode(X, cs.rowmajor, cs.biases, oracle.VARIANT_REFORM)
        Xp = P.pinned_empty(X.shape, np.float32)
        Xp[:] = X
        for devs in ((0, 0), (0, 0, 0)):
            for mode in ("auto", "guarded"):
                plan = P.ExecutionPlan(devices=devs, mode=mode, batch_rows=16_384)
                assert P.encode_dataset(X, cbs, plan).codes.tobytes() == want.tobytes(), (n, devs, mode)
                assert P.encode_dataset_host(Xp, cbs, plan).tobytes() == want.tobytes(), (n, devs, mode)


def test_empty_and_mismatch(P, bulk_setup):
    _, cbs = bulk_setup
    out = P.encode_dataset(np.empty((0, 12), np.float32), cbs, P.ExecutionPlan())
    assert out.n == 0 and out.m == 3
    with pytest.raises(P.ConfigError):
        P.encode_dataset(np.zeros((4, 10), np.float32), cbs, P.ExecutionPlan())


def test_uint16_codes(P):
    rng = np.random.default_rng(33)
    cbs = [P.Codebook.from_rowmajor(0, rng.standard_normal((300, 4)).astype(np.float32))]
    out = P.encode_dataset(rng.standard_normal((10, 4)).astype(np.float32), cbs, P.ExecutionPlan())
    assert out.codes.dtype == np.uint16


# ---- config-shaped parity against the oracle (bit-exact), all modes ----

def _oracle_codes(oracle, X, cs, variant=1):
    return oracle.encode(X, cs.rowmajor, cs.biases, variant)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_parity_vs_oracle(P, oracle, name):
    import torch
    from paper_2605_25521_b200 import configs as C
    cfg = C.CONFIGS[name]
    dev = torch.device("cuda", 0)
    n = 20_000
    X = C.generate(cfg, 0, n, dev)
    Xh = X.cpu().numpy()
    rng = np.random.default_rng(7)
    if cfg.codebook == "sampled":
        rm = C.sampled_codebooks(cfg, Xh.astype(np.float32))
    else:  # codebooks = data subvectors + small jitter: many near-ties
        rows = Xh[rng.choice(n, cfg.k, replace=False)].astype(np.float32)
        rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
        rm = rm + rng.normal(0, 1e-3, rm.shape).astype(np.float32) * (rm.std() + 1e-6)
    cs = cset_of(P, rm)
    want = _oracle_codes(oracle, Xh, cs)
    for mode in MODES:
        got = device_codes(P, Xh, cs, P.EncoderVariant.BLOCKED, mode)
        assert got.tobytes() == want.tobytes(), (name, mode, int((got != want).sum()))


def test_adversarial_near_ties(P, oracle):
    # centroids in 1-ulp clusters and queries on bisectors: the guard must
    # flag and the exact fix-up must reproduce the oracle's first-index rule
    rng = np.random.default_rng(99)
    m, k, sub = 4, 256, 8
    base = rng.standard_normal((m, 64, sub)).astype(np.float32)
    rm = np.repeat(base, 4, axis=1)
    rm[:, 1::4] = np.nextafter(rm[:, 1::4], np.float32(np.inf))
    rm[:, 2::4] = np.nextafter(rm[:, 2::4], np.float32(-np.inf))
    cs = cset_of(P, rm)
    X = np.concatenate([rm[:, i].reshape(-1) for i in range(0, k, 3)]).reshape(-1, m * sub)
    mid = 0.5 * (rm[:, 0::4][:, :32] + rm[:, 4::4][:, :32])
    X = np.concatenate([X, mid.transpose(1, 0, 2).reshape(32, m * sub)]).astype(np.float32)
    X = np.concatenate([X, X + rng.normal(0, 1e-6, X.shape).astype(np.float32)]).astype(np.float32)
    want = _oracle_codes(oracle, X, cs)
    for mode in MODES:
        got = device_codes(P, X, cs, P.EncoderVariant.BLOCKED, mode)
        assert got.tobytes() == want.tobytes(), (mode, int((got != want).sum()))


def test_u8_input_matches_widened_f32(P, oracle):
    rng = np.random.default_rng(4)
    X = rng.integers(0, 256, size=(5000, 128), dtype=np.uint8)
    rm = rng.uniform(0, 255, size=(32, 256, 4)).astype(np.float32)
    cs = cset_of(P, rm)
    want = _oracle_codes(oracle, X.astype(np.float32), cs)
    for mode in MODES:
        assert device_codes(P, X, cs, P.EncoderVariant.BLOCKED, mode).tobytes() == want.tobytes()
    assert P.encode_dataset(X, cs).codes.tobytes() == want.tobytes()


def test_ranking_equivalence_1e6(P, oracle):
    # test_kernels.py:207-231 at >= 1e6 trials: REFERENCE vs REFORMULATED
    # disagreements must be near-ties (gap <= 1e-5 * max(1, d))
    rng = np.random.default_rng(42)
    X = rng.standard_normal((100_000, 160)).astype(np.float32)
    rm = rng.standard_normal((10, 256, 16)).astype(np.float32)
    cs = cset_of(P, rm)
    ref = device_codes(P, X, cs, P.EncoderVariant.REFERENCE)
    ref_or = _oracle_codes(oracle, X, cs, variant=0)
    assert ref.tobytes() == ref_or.tobytes()
    ref2 = device_codes(P, X, cs, P.EncoderVariant.REFORMULATED)
    n, near, fail, _ = oracle.classify_mismatches(X, rm, ref, ref2, 1e-5)
    assert fail == 0 and n * 1.0 / ref.size <= 1e-4


def test_full_size_properties_c3_slice(P, oracle):
    """Size-independent checks at a large N: codes of a 2M-row block are
    identical to the codes of the same rows encoded in 17 uneven pieces,
    and a random sample of rows matches the oracle bit for bit."""
    import torch
    from paper_2605_25521_b200 import configs as C
    cfg = C.CONFIGS["c3"]
    dev = torch.device("cuda", 0)
    n = 2_000_000
    X = C.generate(cfg, 0, n, dev)
    rng = np.random.default_rng(3)
    rm = rng.standard_normal((cfg.m, cfg.k, cfg.sub)).astype(np.float32) * np.float32(0.15)
    cs = cset_of(P, rm)
    full = P.encode_dataset_device(X, cs)
    cuts = np.sort(rng.choice(np.arange(1, n), 16, replace=False))
    parts = [P.encode_dataset_device(X[a:b], cs) for a, b in zip([0, *cuts], [*cuts, n])]
    assert torch.equal(full, torch.cat(parts))
    idx = np.sort(rng.choice(n, 20_000, replace=False))
    sel = X[torch.from_numpy(idx).to(dev)].cpu().numpy()
    assert full[torch.from_numpy(idx).to(dev)].cpu().numpy().tobytes() == _oracle_codes(oracle, sel, cs).tobytes()


def test_device_output_validation(P):
    import torch
    rng = np.random.default_rng(3)
    rm = rng.standard_normal((2, 256, 4)).astype(np.float32)
    cbs = [P.Codebook.from_rowmajor(j, rm[j]) for j in range(2)]
    X = torch.from_numpy(rng.standard_normal((10, 8)).astype(np.float32)).cuda()
    with pytest.raises(P.ConfigError, match="out must be"):
        P.encode_dataset_device(X, cbs, out=torch.empty((10, 3), dtype=torch.uint8, device="cuda"))
    with pytest.raises(P.ConfigError, match="out must be"):
        P.encode_dataset_device(X, cbs, out=torch.empty((10, 2), dtype=torch.int32, device="cuda"))
    with pytest.raises(P.ConfigError, match="best must be"):
        P.encode_dataset_device(X, cbs, best=torch.empty((10, 2), dtype=torch.float64, device="cuda"))
    with pytest.raises(P.ConfigError, match="only produced by the tensor-core path"):
        P.encode_dataset_device(X, cbs, P.ExecutionPlan(mode="exact"),
                                best=torch.empty((10, 2), dtype=torch.float32, device="cuda"))
    out = torch.empty((10, 2), dtype=torch.uint8, device="cuda")
    assert P.encode_dataset_device(X, cbs, out=out) is out
