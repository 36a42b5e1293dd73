"""evaluation.py on the GPU against the reference's own outputs
(tests/golden/eval_golden.npz) and its pkg/tests/test_evaluation.py cases."""

import numpy as np
import pytest

from conftest import golden

EV = golden("eval_golden.npz")
CASES = ["e_s8", "e_s4_ties", "e_k1000", "e_s16"]


@pytest.fixture(scope="module")
def P():
    import paper_2605_25521_b200 as P
    return P


def cbs_of(P, rm):
    return [P.Codebook.from_rowmajor(j, rm[j]) for j in range(rm.shape[0])]


def codes_of(P, name):
    c = EV[f"{name}/codes"]
    return P.PQCodes(codes=c, k=EV[f"{name}/rowmajor"].shape[1])


# ---- CPU: host helpers ----

@pytest.mark.parametrize("name", CASES)
def test_reconstruct_row_matches_reference(P, name):
    cbs = cbs_of(P, EV[f"{name}/rowmajor"])
    got = P.reconstruct(EV[f"{name}/codes"][7], cbs)
    assert got.dtype == np.float32 and got.tobytes() == EV[f"{name}/recon7"].tobytes()


def test_reconstruct_errors_and_report_validation(P):
    cbs = [P.Codebook.from_rowmajor(0, np.array([[1.0, 0.0]], np.float32))]
    with pytest.raises(P.CorruptionError):
        P.reconstruct([5], cbs)
    with pytest.raises(P.ConfigError):
        P.reconstruct([0, 0], cbs)
    with pytest.raises(P.DataError):
        P.EvalReport(mse=1.0, recall_at_n=1.5, top_n=1, n_queries=1, n_db=1, variant="blocked")
    with pytest.raises(P.DataError):
        P.EvalReport(mse=-1.0, recall_at_n=0.5, top_n=1, n_queries=1, n_db=1, variant="blocked")


# ---- GPU ----

@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_tables_and_scores_match_reference(P, name):
    from paper_2605_25521_b200 import evaluation as E
    cbs = cbs_of(P, EV[f"{name}/rowmajor"])
    Q = EV[f"{name}/Q"]
    T = E.adc_tables(Q[0], cbs)
    want = EV[f"{name}/tables0"]
    if EV[f"{name}/rowmajor"].shape[2] <= 12:
        assert T.tobytes() == want.tobytes()  # numpy einsum's summation order reproduced
    else:  # sub > 12: numpy's SIMD order is not modelled -- one rounding apart
        np.testing.assert_allclose(T, want, rtol=4e-7, atol=0)
    codes = codes_of(P, name)
    assert E.adc_scores(want, codes).tobytes() == EV[f"{name}/scores0"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_adc_search_matches_reference(P, name):
    cbs = cbs_of(P, EV[f"{name}/rowmajor"])
    codes = codes_of(P, name)
    idx, dist = P.adc_search_batched(EV[f"{name}/Q"], codes, cbs, 10)
    if EV[f"{name}/rowmajor"].shape[2] <= 12:
        assert np.array_equal(idx, EV[f"{name}/adc_idx"])
        assert dist.tobytes() == EV[f"{name}/adc_dist"].tobytes()
    else:
        assert (idx == EV[f"{name}/adc_idx"]).mean() > 0.95
    i0, d0 = P.adc_search(EV[f"{name}/Q"][3], codes, cbs, 10)
    assert np.array_equal(i0, idx[3]) and np.array_equal(d0, dist[3])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_ground_truth_mse_recall_match_reference(P, name):
    cbs = cbs_of(P, EV[f"{name}/rowmajor"])
    codes = codes_of(P, name)
    X, Q = EV[f"{name}/X"], EV[f"{name}/Q"]
    assert np.array_equal(P.exact_topn(Q, X, 10), EV[f"{name}/gt"])
    assert P.mse_of(X, codes, cbs) == pytest.approx(float(EV[f"{name}/mse"]), rel=1e-12)
    rep = P.evaluate(X, Q, cbs, topn=10, codes=codes)
    if EV[f"{name}/rowmajor"].shape[2] <= 12:
        assert rep.recall_at_n == float(EV[f"{name}/recall"])
    assert rep.n_db == X.shape[0] and rep.n_queries == Q.shape[0] and rep.top_n == 10


@pytest.mark.gpu
def test_reference_adc_cases(P):
    """pkg/tests/test_evaluation.py::TestADC / TestExactTopN restated."""
    rng = np.random.default_rng(43)
    cbs = [P.Codebook.from_rowmajor(j, rng.standard_normal((4, 2)).astype(np.float32)) for j in range(2)]
    db = np.stack([np.concatenate([cbs[0].centroids_rowmajor[a], cbs[1].centroids_rowmajor[b]])
                   for a in range(4) for b in range(4)])
    codes = P.encode_dataset(db, cbs)
    idx, dist = P.adc_search(db[9], codes, cbs, 3)
    assert idx[0] == 9 and dist[0] == 0.0
    one = [P.Codebook.from_rowmajor(0, np.array([[0.5, 0.5]], np.float32))]
    idx, dist = P.adc_search([1.0, 1.0], P.PQCodes(codes=np.zeros((7, 1), np.uint8), k=1), one, 4)
    assert idx.tolist() == [0, 1, 2, 3] and np.all(dist == dist[0])
    two = [P.Codebook.from_rowmajor(0, np.array([[0.0, 0.0], [1.0, 1.0]], np.float32))]
    idx, _ = P.adc_search([0.0, 0.0], P.PQCodes(codes=np.zeros((3, 1), np.uint8), k=2), two, 50)
    assert len(idx) == 3
    gt = P.exact_topn(np.array([[1.0, 0.0]], np.float32), np.array([[1, 0], [0, 1], [1, 0]], np.float32), 3)
    assert gt[0].tolist() == [0, 2, 1]
    rng = np.random.default_rng(46)
    db = rng.standard_normal((200, 8)).astype(np.float32)
    q = rng.standard_normal((5, 8)).astype(np.float32)
    gt = P.exact_topn(q, db, 7)
    for i in range(5):
        d = ((db.astype(np.float64) - q[i].astype(np.float64)) ** 2).sum(axis=1)
        assert gt[i].tolist() == np.lexsort((np.arange(200), d))[:7].tolist()


@pytest.mark.gpu
def test_evaluate_variant_irrelevance_and_errors(P):
    ds = P.synth_dataset(2000, 32, 16, seed=47)
    queries = ds.data[:100]
    cbs = P.train_all_codebooks(ds, P.PQParams(d=32, m=4, k=64), P.TrainConfig(k=64, seed=47))
    reps = {v: P.evaluate(ds, queries, cbs, variant=v, topn=10) for v in P.EncoderVariant}
    assert len({(r.mse, r.recall_at_n) for r in reps.values()}) == 1
    assert P.evaluate(ds, queries, cbs, topn=1).recall_at_n >= 0.9
    rep = P.evaluate(ds, queries, cbs, topn=5)
    assert rep.n_db == 2000 and rep.n_queries == 100 and rep.top_n == 5 and rep.variant == "blocked"
    with pytest.raises(P.DataError):
        P.evaluate(ds, np.empty((0, 32), np.float32), cbs)


@pytest.mark.gpu
def test_topn_large_database_and_nan(P):
    """Selection over a 3M-row database with planted ties and NaN scores."""
    import torch
    from paper_2605_25521_b200 import evaluation as E
    rng = np.random.default_rng(8)
    n = 3_000_000
    v = rng.random((2, n)).astype(np.float32)
    v[0, [5, 17, 2_999_999]] = 1e-9        # ties at the minimum -> index order
    v[1, :1000] = np.nan                    # NaN sorts last
    v[1, 123_456] = -1.0
    idx, val = E._topn_dev(torch.from_numpy(v).cuda(), 20, torch.device("cuda", 0))
    for r in range(2):
        want = np.lexsort((np.arange(n), v[r]))[:20]
        assert idx[r].cpu().numpy().tolist() == want.tolist()
        assert np.array_equal(val[r].cpu().numpy(), v[r][want], equal_nan=True)
