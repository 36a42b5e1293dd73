"""The reference's verification / ablation harness (cli.py run_verify,
run_bench_matrix, BenchResult; exercised by pkg/tests/test_acceptance.py
criterion 5) mirrored on the GPU path."""

import csv

import numpy as np
import pytest

import paper_2605_25521_b200 as P


def test_bench_result_row_format(tmp_path):
    r = P.BenchResult(variant="blocked+reform", order=P.CHUNK_MAJOR, w=16, block_size=4096, n=10, d=8, m=2,
                      k=256, wall_seconds=0.5, vectors_per_second=20.0, speedup_vs_baseline=3.25)
    assert r.csv_row() == ["blocked+reform", "chunk_major", 16, 4096, 10, 8, 2, 256, "0.500000", "20.0", "3.2500"]
    path = tmp_path / "bench.csv"
    P.write_bench_csv([r, r], path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == P.BENCH_CSV_COLUMNS
    assert len(rows) == 3 and rows[1] == [str(v) for v in r.csv_row()]


def test_harness_needs_cuda(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    cb = P.Codebook.from_rowmajor(0, np.eye(4, dtype=np.float32))
    with pytest.raises(P.NativeUnavailable):
        P.run_verify(np.zeros((3, 4), np.float32), [cb], samples=3, tolerance=1e-5)
    with pytest.raises(P.NativeUnavailable):
        P.run_bench_matrix(np.zeros((3, 4), np.float32), [cb], reps=1)


def _near_tie_data(n=4000, m=4, k=256, sub=8, seed=3):
    rng = np.random.default_rng(seed)
    rm = np.round(rng.uniform(0, 255, (m, k, sub))).astype(np.float32)
    # rows on the bisector of centroid pairs make REFERENCE and REFORMULATED disagree at near-ties
    X = np.empty((n, m * sub), np.float32)
    for j in range(m):
        a = rng.integers(0, k, n)
        b = rng.integers(0, k, n)
        mid = 0.5 * (rm[j, a] + rm[j, b])  # half-integers: exact float32 bisectors (ties)
        mid[1::2] += rng.normal(0, 1e-4, (n // 2, sub))
        X[:, j * sub:(j + 1) * sub] = mid
    return X, [P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)]


def test_verify_golden_inputs_regenerate():
    import zlib
    from conftest import golden
    g = golden("verify_golden.npz")
    X, cbs = _near_tie_data()
    assert zlib.crc32(X.tobytes()) == int(g["v/X_crc32"])
    assert np.stack([cb.centroids_rowmajor for cb in cbs]).tobytes() == g["v/rowmajor"].tobytes()


def test_oracle_reproduces_reference_verify(oracle):
    """The oracle's REFERENCE / REFORMULATED codes disagree exactly where the
    reference's run_verify found disagreements, with the same codes."""
    from conftest import golden
    g = golden("verify_golden.npz")
    X, cbs = _near_tie_data()
    cs = P.CodebookSet.from_codebooks(cbs)
    rng = np.random.Generator(np.random.PCG64(7))
    Xs = np.ascontiguousarray(X[np.sort(rng.choice(X.shape[0], size=3000, replace=False))])
    ref = oracle.encode(Xs, cs.rowmajor, cs.biases, oracle.VARIANT_REFERENCE)
    form = oracle.encode(Xs, cs.rowmajor, cs.biases, oracle.VARIANT_REFORM)
    ij = np.argwhere(ref != form)
    assert ij.tolist() == g["v/ij"].tolist()
    assert np.stack([ref[tuple(ij.T)], form[tuple(ij.T)], form[tuple(ij.T)]], 1).tolist() == g["v/codes"].tolist()


@pytest.mark.gpu
def test_run_verify_matches_reference():
    """cli.run_verify of the reference on the same seeded data
    (tests/golden/verify_golden.npz): the same sample, the same disagreements,
    codes, gaps and near-tie / failure split."""
    from conftest import golden
    g = golden("verify_golden.npz")
    X, cbs = _near_tie_data()
    checked, near, fail, details = P.run_verify(X, cbs, samples=3000, tolerance=1e-5, seed=7)
    assert [checked, near, fail] == g["v/counts"].tolist()
    assert [(i, j) for i, j, *_ in details] == [tuple(r) for r in g["v/ij"].tolist()]
    assert [kind == "near-tie" for _, _, kind, _, _ in details] == g["v/near"].tolist()
    assert [gap for _, _, _, gap, _ in details] == g["v/gap"].tolist()
    assert [[c["REFERENCE"], c["REFORMULATED"], c["BLOCKED"]] for *_, c in details] == g["v/codes"].tolist()


@pytest.mark.gpu
def test_run_bench_matrix_rows(tmp_path):
    X, cbs = _near_tie_data(n=20000)
    res = P.run_bench_matrix(X, cbs, w=16, reps=1)
    assert [(r.variant, r.order) for r in res] == [
        ("reference", P.VECTOR_MAJOR), ("blocked", P.VECTOR_MAJOR), ("blocked", P.CHUNK_MAJOR),
        ("blocked+reform", P.CHUNK_MAJOR)]
    assert res[0].speedup_vs_baseline == 1.0
    for r in res:
        assert r.n == 20000 and r.d == 32 and r.m == 4 and r.k == 256 and r.w == 16
        assert r.wall_seconds > 0 and r.vectors_per_second > 0
    P.write_bench_csv(res, tmp_path / "m.csv")
    assert len(open(tmp_path / "m.csv").read().splitlines()) == 5


def test_einsum_rowsq_is_numpys_order():
    """run_verify's gaps use np.einsum("kt,kt->k")'s float64 order (cli.py:194-201)."""
    from paper_2605_25521_b200.harness import einsum_rowsq
    rng = np.random.default_rng(0)
    for s in range(1, 20):
        d = rng.standard_normal((20, 9, s)) * 10.0 ** rng.integers(-3, 4)
        want = np.stack([np.einsum("kt,kt->k", d[q], d[q]) for q in range(20)])
        assert einsum_rowsq(d).tobytes() == want.tobytes()
