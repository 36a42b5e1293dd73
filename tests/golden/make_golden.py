"""Generate the golden vectors that pin the oracle (and, through it, the GPU
path) to the reference implementation.

Run HERE (the container that has /root/reference), never on the GPU box:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py
    # full-size Lloyd subspaces (samples dumped on the GPU box first):
    gpurun -- python scripts/dump_train_samples.py
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py full gpurun_out/train_samples.npz

It imports the reference package ``cspq`` (read-only, untouched) and records
its outputs on small seeded inputs into ``tests/golden/*.npz``.  The inputs
mirror the reference's own hot-path tests (pkg/tests/test_kernels.py,
test_bulk.py, test_training.py, test_acceptance.py) plus config-shaped cases
(BASELINE.json configs 1-5 at reduced N).  Only the generated .npz files and
this script are committed; nothing here is imported at test time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    import cspq  # noqa: F401
    from cspq import bulk, core, kernels, training
    return bulk, core, kernels, training


def encode_cases(bulk, core, kernels):
    EV = kernels.EncoderVariant
    rng = np.random.default_rng(20260101)
    out = {}

    def put(name, X, rowmajor, in_u8=False):
        cbs = [core.Codebook.from_rowmajor(j, rowmajor[j]) for j in range(rowmajor.shape[0])]
        cset = bulk.CodebookSet.from_codebooks(cbs)
        out[f"{name}/X"] = X
        out[f"{name}/rowmajor"] = cset.rowmajor
        out[f"{name}/biases"] = cset.biases
        for var in (EV.REFERENCE, EV.REFORMULATED, EV.BLOCKED):
            codes = bulk.encode_dataset(X, cset, bulk.ExecutionPlan(variant=var, w=16)).codes
            out[f"{name}/codes_{var.value}"] = codes
        out[f"{name}/codes_nobias"] = bulk.encode_dataset(
            X, cset, bulk.ExecutionPlan(variant=EV.BLOCKED, w=8), precomputed_bias=False).codes
        # winning scores (bitwise) for the first rows, via the per-subvector API
        nb = min(64, X.shape[0])
        sub = cset.sub_dim
        best_reform = np.zeros((nb, cset.m), np.float32)
        best_ref = np.zeros((nb, cset.m), np.float32)
        for i in range(nb):
            for j in range(cset.m):
                v = np.asarray(X[i, j * sub:(j + 1) * sub], dtype=np.float32)
                best_reform[i, j] = kernels.encode_reform_with_score(v, cset[j])[1]
                best_ref[i, j] = kernels.encode_ref_with_score(v, cset[j])[1]
        out[f"{name}/best_reformulated"] = best_reform
        out[f"{name}/best_reference"] = best_ref

    # random normal, generic shapes (test_kernels-style)
    put("rand_m4_k256_s8", rng.standard_normal((3000, 32)).astype(np.float32),
        rng.standard_normal((4, 256, 8)).astype(np.float32))
    # remainder blocks / small k / odd sub (test_kernels.py:90-97)
    put("rand_m3_k5_s4", rng.standard_normal((500, 12)).astype(np.float32),
        rng.standard_normal((3, 5, 4)).astype(np.float32))
    put("rand_m2_k7_s3", rng.standard_normal((500, 6)).astype(np.float32),
        rng.standard_normal((2, 7, 3)).astype(np.float32))
    put("rand_m1_k1_s6", rng.standard_normal((50, 6)).astype(np.float32),
        rng.standard_normal((1, 1, 6)).astype(np.float32))
    put("rand_m4_k33_s7", rng.standard_normal((500, 28)).astype(np.float32),
        rng.standard_normal((4, 33, 7)).astype(np.float32))
    put("rand_m2_k37_s16", rng.standard_normal((500, 32)).astype(np.float32),
        rng.standard_normal((2, 37, 16)).astype(np.float32))
    put("rand_m5_k64_s1", rng.standard_normal((400, 5)).astype(np.float32),
        rng.standard_normal((5, 64, 1)).astype(np.float32))
    put("rand_m3_k256_s2", rng.standard_normal((600, 6)).astype(np.float32),
        rng.standard_normal((3, 256, 2)).astype(np.float32))
    # uint16 codes (test_bulk.py:74-78)
    put("rand_m2_k300_s4", rng.standard_normal((400, 8)).astype(np.float32),
        rng.standard_normal((2, 300, 4)).astype(np.float32))
    put("rand_m1_k1000_s8", rng.standard_normal((200, 8)).astype(np.float32),
        rng.standard_normal((1, 1000, 8)).astype(np.float32))
    # large dynamic range
    put("scaled_m4_k256_s8", (rng.standard_normal((1000, 32)) * 1e3).astype(np.float32),
        (rng.standard_normal((4, 256, 8)) * 1e3).astype(np.float32))
    # config-1-like: integer data, codebook = distinct data subvectors (tie-heavy)
    cent = rng.uniform(0, 255, size=(8, 128))
    lab = rng.integers(0, 8, size=3000)
    X1 = np.clip(np.rint(cent[lab] + rng.normal(0, 20, size=(3000, 128))), 0, 255).astype(np.float32)
    rm = np.zeros((16, 256, 8), np.float32)
    for j in range(16):
        u = np.unique(X1[:, j * 8:(j + 1) * 8], axis=0)
        rm[j] = u[rng.choice(u.shape[0], 256, replace=False)]
    put("c1like_m16_k256_s8", X1, rm)
    # config-4-like: uint8 input widened in the encoder, d_sub = 4
    X4 = np.clip(np.rint(cent[lab][:, :128] + rng.normal(0, 15, size=(3000, 128))), 0, 255).astype(np.uint8)
    rm4 = (rng.uniform(0, 255, size=(32, 256, 4))).astype(np.float32)
    put("c4like_u8_m32_k256_s4", X4, rm4, in_u8=True)
    # unit-normalised rows (configs 3/5)
    X3 = rng.standard_normal((2000, 96)).astype(np.float32)
    X3 /= np.linalg.norm(X3, axis=1, keepdims=True)
    rm3 = rng.standard_normal((12, 256, 8)).astype(np.float32) * np.float32(0.2)
    put("unit_m12_k256_s8", X3.astype(np.float32), rm3)
    # duplicated centroids: exact ties -> smaller index (test_kernels.py:141-151)
    rmt = rng.standard_normal((3, 32, 8)).astype(np.float32)
    rmt[:, 20] = rmt[:, 3]
    rmt[:, 31] = rmt[:, 0]
    Xt = np.concatenate([rmt[0, [3, 0, 20, 31]].reshape(4, 8)] * 3, axis=1)
    Xt = np.concatenate([Xt, rng.standard_normal((60, 24)).astype(np.float32)]).astype(np.float32)
    put("ties_m3_k32_s8", Xt, rmt)
    # non-finite rows: encode_dataset does not validate raw ndarrays
    Xn = rng.standard_normal((40, 16)).astype(np.float32)
    Xn[3, 2] = np.nan
    Xn[5, :] = np.nan
    Xn[7, 9] = np.inf
    Xn[8, 1] = -np.inf
    Xn[9, 0] = np.float32(3e38)
    Xn[10, 12] = np.float32(1e-42)  # denormal
    put("nonfinite_m2_k16_s8", Xn, rng.standard_normal((2, 16, 8)).astype(np.float32))
    # known answers (test_kernels.py:37-88)
    put("hand_blocked", np.array([[1, 0]], np.float32),
        np.array([[[1, 0], [0, 1], [2, 0], [0, 0]]], np.float32))
    put("hand_identity", np.array([[1, 0]], np.float32), np.array([[[3, 4]]], np.float32))
    put("hand_pair", np.array([[0.6, 0.4]], np.float32), np.array([[[1, 0], [0, 1]]], np.float32))
    return out


def lloyd_cases(training):
    TC = training.TrainConfig
    rng = np.random.default_rng(777)
    out = {}

    def put(name, P64, init, iters, tol):
        r = training.lloyd_iterate(P64, init, TC(k=init.shape[0], max_iters=iters, tol=tol))
        out[f"{name}/pts"] = P64.astype(np.float32)
        out[f"{name}/init"] = init
        out[f"{name}/max_iters"] = np.int64(iters)
        out[f"{name}/tol"] = np.float64(tol)
        out[f"{name}/centroids"] = r.centroids
        out[f"{name}/objectives"] = np.asarray(r.objectives, np.float64)
        out[f"{name}/assignments"] = r.assignments
        out[f"{name}/iterations"] = np.int64(r.iterations)

    # empty-cluster repair (test_training.py:142-155)
    P = np.array([[0.0], [0.1], [0.2], [10.0], [10.1], [50.0]], np.float32).astype(np.float64)
    put("repair_1d", P, np.array([[0.0], [0.0], [10.0]]), 10, 1e-4)
    # gaussian blobs, tol stop
    means = rng.uniform(-5, 5, size=(16, 2))
    P = (means[rng.integers(0, 16, 4000)] + rng.normal(0, 0.4, (4000, 2))).astype(np.float32).astype(np.float64)
    put("blobs_k16_s2", P, P[rng.choice(4000, 16, replace=False)], 50, 1e-4)
    # config-2-like (d_sub 8, k 256, sample-point init, tol 0)
    cen = rng.uniform(0, 1, size=(64, 8))
    P = np.clip(cen[rng.integers(0, 64, 12000)] + rng.normal(0, 0.08, (12000, 8)), 0, None)
    P = P.astype(np.float32).astype(np.float64)
    put("c2like_k256_s8", P, P[np.sort(rng.choice(12000, 256, replace=False))], 25, 0.0)
    # config-3-like: unit-normalised embeddings
    Z = rng.standard_normal((8000, 64))
    Z /= np.linalg.norm(Z, axis=1, keepdims=True)
    P = Z[:, 8:16].astype(np.float32).astype(np.float64)
    put("c3like_k256_s8", P, P[np.sort(rng.choice(8000, 256, replace=False))], 10, 0.0)
    # config-4-like: integer data, d_sub 4, duplicates -> empty-cluster repair
    cen = rng.uniform(0, 255, size=(32, 4))
    P = np.clip(np.rint(cen[rng.integers(0, 32, 10000)] + rng.normal(0, 15, (10000, 4))), 0, 255)
    P = P.astype(np.float32).astype(np.float64)
    init = P[np.sort(rng.choice(10000, 256, replace=False))].copy()
    init[5] = init[4]  # guaranteed duplicate -> one empty cluster in iteration 1
    put("c4like_k256_s4", P, init, 20, 0.0)
    # k = 1 mean
    P = np.array([[1.0, 5.0], [3.0, 5.0], [2.0, 8.0]], np.float64)
    put("k1", P, P[:1].copy(), 5, 1e-4)
    return out


def train_cases(core, training):
    """Reference default path (k-means++ seeding, per-subspace sampling)."""
    rng = np.random.default_rng(4242)
    out = {}
    means = rng.uniform(-1, 1, size=(24, 32)).astype(np.float32)
    X = (means[rng.integers(0, 24, 6000)] + rng.normal(0, 0.05, (6000, 32)).astype(np.float32)).astype(np.float32)
    ds = core.VectorDataset(data=np.ascontiguousarray(X))
    params = core.PQParams(d=32, m=4, k=64)
    cfg = training.TrainConfig(k=64, seed=11, sample_cap=3000, max_iters=12)
    cbs, reps = training.train_all_codebooks_report(ds, params, cfg)
    out["kmpp/X"] = X
    out["kmpp/centroids"] = np.stack([cb.centroids_rowmajor for cb in cbs])
    out["kmpp/biases"] = np.stack([cb.biases for cb in cbs])
    for j, r in enumerate(reps):
        out[f"kmpp/objectives_{j}"] = np.asarray(r.objectives)
        out[f"kmpp/assignments_{j}"] = r.assignments
        out[f"kmpp/iterations_{j}"] = np.int64(r.iterations)
    # the seeding alone, for one subspace (training.py:76-92)
    rngs = training._subspace_rngs(11, 4)
    pts = np.ascontiguousarray(X[:, 8:16])
    sampled = training._sample(pts, 3000, rngs[1])
    init = training._kmeanspp_init(sampled.astype(np.float64), 64, rngs[1])
    out["kmpp/seed_init_sub1"] = init
    return out


def pairwise_cases():
    rng = np.random.default_rng(5)
    out = {}
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 8193, 100003):
        a = rng.random(n) * rng.random(n) * 1e3
        out[f"pw/{n}/a"] = a
        out[f"pw/{n}/sum"] = np.float64(a.sum())
    return out


def io_cases():
    """File bytes written by the reference's own writers (io.py) and the
    errors its readers raise, for the format layer and the GPU file encoder."""
    import struct
    import tempfile
    from cspq import bulk, core, io
    out = {}
    rng = np.random.default_rng(20260202)
    tmp = tempfile.mkdtemp()

    def raw(name, path):
        out[name] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8).copy()

    # vector files
    f32 = rng.standard_normal((37, 24)).astype(np.float32)
    u8 = rng.integers(0, 256, (29, 16)).astype(np.uint8)
    i32 = rng.integers(0, 5000, (11, 7)).astype(np.int32)
    io.write_fvecs(os.path.join(tmp, "a.fvecs"), f32)
    io.write_bvecs(os.path.join(tmp, "a.bvecs"), u8)
    io.write_ivecs(os.path.join(tmp, "a.ivecs"), i32)
    out["fvecs/data"], out["bvecs/data"], out["ivecs/data"] = f32, u8, i32
    for ext in ("fvecs", "bvecs", "ivecs"):
        raw(f"{ext}/bytes", os.path.join(tmp, f"a.{ext}"))
    # containers
    cbs = [core.Codebook.from_rowmajor(j, rng.standard_normal((16, 4)).astype(np.float32)) for j in range(3)]
    io.write_codebooks(os.path.join(tmp, "c.pqcb"), cbs)
    raw("pqcb/bytes", os.path.join(tmp, "c.pqcb"))
    out["pqcb/rowmajor"] = np.stack([c.centroids_rowmajor for c in cbs])
    c8 = core.PQCodes(codes=rng.integers(0, 200, (50, 4)).astype(np.uint8), k=200)
    c16 = core.PQCodes(codes=rng.integers(0, 1000, (20, 3)).astype(np.uint16), k=1000)
    io.write_codes(os.path.join(tmp, "c8.pqcd"), c8)
    io.write_codes(os.path.join(tmp, "c16.pqcd"), c16)
    raw("pqcd8/bytes", os.path.join(tmp, "c8.pqcd"))
    raw("pqcd16/bytes", os.path.join(tmp, "c16.pqcd"))
    out["pqcd8/codes"], out["pqcd16/codes"] = c8.codes, c16.codes
    # encode-from-file cases: read_fvecs / read_bvecs + encode_dataset + write_codes
    for name, ext, X, sub in (("file_f32", "fvecs", (rng.standard_normal((3000, 64)) * 3).astype(np.float32), 8),
                              ("file_u8", "bvecs", rng.integers(0, 256, (2500, 32)).astype(np.uint8), 4)):
        m = X.shape[1] // sub
        Xf = X.astype(np.float32)
        rm = np.stack([Xf[rng.choice(X.shape[0], 256, replace=False), j * sub:(j + 1) * sub] for j in range(m)])
        rm = rm + rng.normal(0, 0.25, rm.shape).astype(np.float32)
        cset = bulk.CodebookSet.from_codebooks([core.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
        path = os.path.join(tmp, f"{name}.{ext}")
        (io.write_fvecs if ext == "fvecs" else io.write_bvecs)(path, X)
        ds = (io.read_fvecs if ext == "fvecs" else io.read_bvecs)(path)
        codes = bulk.encode_dataset(ds, cset)
        io.write_codes(os.path.join(tmp, f"{name}.pqcd"), codes)
        out[f"{name}/X"], out[f"{name}/rowmajor"] = X, cset.rowmajor
        raw(f"{name}/vecs_bytes", path)
        raw(f"{name}/pqcd_bytes", os.path.join(tmp, f"{name}.pqcd"))
    # reader errors: (message, offset) for malformed files
    bad = {
        "empty": b"",
        "inconsistent": struct.pack("<i", 2) + struct.pack("<2f", 1, 2) + struct.pack("<i", 3) + struct.pack("<3f", 1, 2, 3),
        "truncated_body": struct.pack("<i", 4) + struct.pack("<2f", 1, 2),
        "truncated_header": struct.pack("<i", 2) + struct.pack("<2f", 1, 2) + b"\x02\x00",
        "nonpositive": struct.pack("<i", 2) + struct.pack("<2f", 1, 2) + struct.pack("<i", -1),
        "nonfinite": struct.pack("<i", 2) + struct.pack("<2f", 1, 2) + struct.pack("<i", 2) + struct.pack("<2f", 3, float("inf")),
    }
    msgs = []
    for key, b in bad.items():
        path = os.path.join(tmp, f"{key}.fvecs")
        open(path, "wb").write(b)
        try:
            io.read_fvecs(path)
            msgs.append((key, "", -1))
        except core.FormatError as e:
            msgs.append((key, str(e).replace(path, "<path>"), -1 if e.offset is None else e.offset))
        out[f"err/{key}/bytes"] = np.frombuffer(b, dtype=np.uint8).copy()
    out["err/keys"] = np.array([k for k, _, _ in msgs])
    out["err/messages"] = np.array([msg for _, msg, _ in msgs])
    out["err/offsets"] = np.array([o for _, _, o in msgs], dtype=np.int64)
    # synth_dataset bits
    out["synth/data"] = io.synth_dataset(64, 12, 5, seed=7).data
    return out


def eval_cases():
    """Reference evaluation.py outputs: tables / scores bits, ADC top-N, exact
    ground truth, mse_of and evaluate() reports."""
    from cspq import bulk, core, evaluation as ev
    out = {}
    rng = np.random.default_rng(20260303)
    cases = []
    # (name, n, d, m, k, dup): dup > 0 duplicates rows to force exact score / distance ties
    for name, n, m, sub, k, dup in (("e_s8", 3000, 8, 8, 256, 0), ("e_s4_ties", 2000, 8, 4, 64, 400),
                                    ("e_k1000", 1500, 4, 8, 1000, 0), ("e_s16", 1200, 2, 16, 256, 0)):
        d = m * sub
        X = rng.standard_normal((n, d)).astype(np.float32)
        if dup:
            X[-dup:] = X[:dup]
        Q = np.concatenate([rng.standard_normal((14, d)).astype(np.float32), X[:6] + 0.0]).astype(np.float32)
        rm = np.stack([X[rng.choice(n, k, replace=k > n), j * sub:(j + 1) * sub] for j in range(m)])
        rm = (rm + rng.normal(0, 0.05, rm.shape)).astype(np.float32)
        cbs = [core.Codebook.from_rowmajor(j, rm[j]) for j in range(m)]
        codes = bulk.encode_dataset(X, bulk.CodebookSet.from_codebooks(cbs))
        out[f"{name}/X"], out[f"{name}/Q"], out[f"{name}/rowmajor"], out[f"{name}/codes"] = X, Q, rm, codes.codes
        out[f"{name}/tables0"] = ev.adc_tables(Q[0], cbs)
        out[f"{name}/scores0"] = ev.adc_scores(out[f"{name}/tables0"], codes)
        idx, dist = zip(*[ev.adc_search(q, codes, cbs, 10) for q in Q])
        out[f"{name}/adc_idx"], out[f"{name}/adc_dist"] = np.stack(idx), np.stack(dist)
        out[f"{name}/gt"] = ev.exact_topn(Q, X, 10)
        out[f"{name}/mse"] = np.float64(ev.mse_of(X, codes, cbs))
        rep = ev.evaluate(core.VectorDataset(data=X), core.VectorDataset(data=Q), cbs, topn=10, codes=codes)
        out[f"{name}/recall"] = np.float64(rep.recall_at_n)
        out[f"{name}/recon7"] = ev.reconstruct(codes.codes[7], cbs)
    return out


def verify_cases():
    """Reference cli.run_verify (three-way encoder equivalence with the float64
    near-tie classifier) on bisector-heavy data where REFERENCE and
    REFORMULATED disagree."""
    from cspq import bulk, core
    from cspq.cli import run_verify
    out = {}
    rng = np.random.default_rng(3)
    n, m, k, sub = 4000, 4, 256, 8
    rm = np.round(rng.uniform(0, 255, (m, k, sub))).astype(np.float32)
    X = np.empty((n, m * sub), np.float32)
    for j in range(m):
        a = rng.integers(0, k, n)
        b = rng.integers(0, k, n)
        mid = 0.5 * (rm[j, a] + rm[j, b])  # half-integers: exact float32 bisectors (ties)
        mid[1::2] += rng.normal(0, 1e-4, (n // 2, sub))
        X[:, j * sub:(j + 1) * sub] = mid
    cbs = [core.Codebook.from_rowmajor(j, rm[j]) for j in range(m)]
    # (a VectorDataset: the reference's hasattr(dataset, "data") probe breaks on raw arrays)
    checked, near, fail, details = run_verify(core.VectorDataset(data=X), cbs, 3000, 1e-5, seed=7)
    import zlib
    out["v/X_crc32"], out["v/rowmajor"] = np.int64(zlib.crc32(X.tobytes())), rm  # X is regenerated by the test
    out["v/counts"] = np.array([checked, near, fail], np.int64)
    out["v/ij"] = np.array([(i, j) for i, j, *_ in details], np.int64).reshape(-1, 2)
    out["v/near"] = np.array([kind == "near-tie" for _, _, kind, _, _ in details], bool)
    out["v/gap"] = np.array([gap for _, _, _, gap, _ in details], np.float64)
    out["v/codes"] = np.array([[c["REFERENCE"], c["REFORMULATED"], c["BLOCKED"]] for *_, c in details],
                              np.int64).reshape(-1, 3)
    return out


def full_lloyd_cases(training, samples_path):
    """The reference's own lloyd_iterate (training.py:109-159, tol 0, the
    config's sample-point init) on full-size training-sample subspaces of
    BASELINE configs 2-5: c2 100K x 8 / 25 iterations, c3 200K x 8 / 10,
    c4 1M x 4 / 20, c5 100K x 8 / 10.  The samples are generated on the GPU
    (paper_2605_25521_b200/configs.py, Philox) and dumped by
    scripts/dump_train_samples.py; only their SHA-256 is committed, and the
    -m gpu test regenerates them and checks the hash before comparing."""
    from paper_2605_25521_b200 import configs as C
    S = np.load(samples_path)
    out = {}
    for key in sorted(k for k in S.files if k.endswith("/points")):
        name, j, _ = key.split("/")
        cfg = C.CONFIGS[name]
        pts = S[key]
        init = S[f"{name}/{j}/init"]
        assert pts.shape == (cfg.n_train, cfg.sub) and init.shape == (cfg.k, cfg.sub)
        tc = training.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
        r = training.lloyd_iterate(pts.astype(np.float64), init.astype(np.float64), tc)
        g = f"{name}/{j}"
        out[f"{g}/points_sha256"] = S[f"{g}/points_sha256"]
        out[f"{g}/sample_sha256"] = S[f"{name}/sample_sha256"]
        out[f"{g}/init"] = init
        out[f"{g}/centroids"] = r.centroids
        out[f"{g}/objectives"] = np.asarray(r.objectives, np.float64)
        out[f"{g}/assignments"] = r.assignments.astype(np.uint8)  # k = 256
        out[f"{g}/iterations"] = np.int64(r.iterations)
        print(g, r.iterations, r.objectives[-1], flush=True)
    return out


def kpp_zero_mass_cases(training):
    """_kmeanspp_init (training.py:76-92) when D^2 mass runs out: fewer distinct points than
    k, so from some step on total == 0 and the reference draws rng.integers(n) instead of
    rng.choice.  Records the seeds and the next draw of the generator afterwards."""
    out = {}
    rng0 = np.random.default_rng(20261020)
    for case, (n, ndist, k, sub, seed) in enumerate([(50, 3, 8, 2, 5), (400, 17, 64, 4, 9), (33, 1, 4, 3, 1)]):
        base = rng0.standard_normal((ndist, sub))
        pts = base[rng0.integers(0, ndist, n)]
        pts[:ndist] = base  # every distinct row present
        rng = np.random.default_rng(seed)
        init = training._kmeanspp_init(pts.astype(np.float64), k, rng)
        g = f"z{case}"
        out[f"{g}/pts"] = pts
        out[f"{g}/k"] = np.int64(k)
        out[f"{g}/seed"] = np.int64(seed)
        out[f"{g}/init"] = init
        out[f"{g}/next_draw"] = np.int64(rng.integers(1 << 30))
    return out


def main():
    if sys.argv[1:2] == ["kppzero"]:
        _, _, _, training = _ref()
        np.savez_compressed(os.path.join(HERE, "kpp_zero_golden.npz"), **kpp_zero_mass_cases(training))
        return
    if sys.argv[1:2] == ["full"]:  # full-size Lloyd goldens: make_golden.py full <train_samples.npz>
        sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
        _, _, _, training = _ref()
        np.savez_compressed(os.path.join(HERE, "lloyd_full_golden.npz"), **full_lloyd_cases(training, sys.argv[2]))
        return
    bulk, core, kernels, training = _ref()
    if sys.argv[1:] == ["verify"]:  # (added later: regenerate only this archive)
        np.savez_compressed(os.path.join(HERE, "verify_golden.npz"), **verify_cases())
        return
    np.savez_compressed(os.path.join(HERE, "encode_golden.npz"), **encode_cases(bulk, core, kernels))
    np.savez_compressed(os.path.join(HERE, "lloyd_golden.npz"), **lloyd_cases(training))
    np.savez_compressed(os.path.join(HERE, "train_golden.npz"), **train_cases(core, training))
    np.savez_compressed(os.path.join(HERE, "pairwise_golden.npz"), **pairwise_cases())
    np.savez_compressed(os.path.join(HERE, "io_golden.npz"), **io_cases())
    np.savez_compressed(os.path.join(HERE, "eval_golden.npz"), **eval_cases())
    np.savez_compressed(os.path.join(HERE, "verify_golden.npz"), **verify_cases())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
