"""Pin the CPU oracle to the reference: every golden vector recorded from the
reference package (tests/golden/make_golden.py) must be reproduced --
bit-exactly for encode, to summation-order tolerance for Lloyd."""

import numpy as np
import pytest

from conftest import cases, golden, group

ENC = golden("encode_golden.npz")
LLOYD = golden("lloyd_golden.npz")
PW = golden("pairwise_golden.npz")


@pytest.mark.parametrize("case", cases(ENC))
def test_encode_bitexact(oracle, case):
    g = group(ENC, case)
    for variant, key in ((oracle.VARIANT_REFERENCE, "codes_reference"),
                         (oracle.VARIANT_REFORM, "codes_reformulated"),
                         (oracle.VARIANT_REFORM, "codes_blocked"),
                         (oracle.VARIANT_NOBIAS, "codes_nobias")):
        got = oracle.encode(g["X"], g["rowmajor"], g["biases"], variant)
        assert got.dtype == g[key].dtype
        assert got.tobytes() == g[key].tobytes(), (case, key)


@pytest.mark.parametrize("case", cases(ENC))
def test_encode_scores_bitwise(oracle, case):
    g = group(ENC, case)
    nb = g["best_reformulated"].shape[0]
    _, best = oracle.encode(g["X"][:nb], g["rowmajor"], g["biases"], oracle.VARIANT_REFORM, want_best=True)
    assert best.tobytes() == g["best_reformulated"].tobytes()
    _, best = oracle.encode(g["X"][:nb], g["rowmajor"], g["biases"], oracle.VARIANT_REFERENCE, want_best=True)
    assert best.tobytes() == g["best_reference"].tobytes()


@pytest.mark.parametrize("case", cases(ENC))
def test_biases_bitexact(oracle, case):
    g = group(ENC, case)
    assert oracle.compute_biases(g["rowmajor"]).tobytes() == g["biases"].tobytes()


@pytest.mark.parametrize("case", cases(LLOYD))
def test_lloyd_matches_reference(oracle, case):
    g = group(LLOYD, case)
    r = oracle.lloyd(g["pts"].astype(np.float64), g["init"], int(g["max_iters"]), float(g["tol"]))
    assert r["iterations"] == int(g["iterations"])
    assert np.array_equal(r["assignments"], g["assignments"])
    # float64 norms in np.einsum's order (oracle_einsum_dot) and the dot as an ascending fused
    # chain: centroids and every objective equal the reference's bit for bit
    assert r["centroids"].tobytes() == g["centroids"].tobytes()
    objs = np.asarray(r["objectives"])
    assert objs.shape == g["objectives"].shape
    assert objs.tobytes() == g["objectives"].tobytes()


@pytest.mark.parametrize("n", list(range(1, 25)) + [31, 64, 100])
def test_einsum_dot_is_numpys(oracle, n):
    """oracle_einsum_dot reproduces np.einsum("it,it->i") / ("kt,kt->k") on float64 rows --
    the order of training.py:61/70/88/134/154 -- bit for bit (numpy of this image)."""
    rng = np.random.default_rng(n)
    for scale in (1.0, 1e-3, 1e5):
        a = rng.standard_normal((300, n)) * scale
        b = rng.standard_normal((300, n))
        want_aa = np.einsum("it,it->i", a, a)
        want_ab = np.einsum("kt,kt->k", a, b)
        got_aa = np.array([oracle.einsum_dot(r, r) for r in a])
        got_ab = np.array([oracle.einsum_dot(r, q) for r, q in zip(a, b)])
        assert got_aa.tobytes() == want_aa.tobytes()
        assert got_ab.tobytes() == want_ab.tobytes()


@pytest.mark.parametrize("n", sorted({int(k.split("/")[1]) for k in PW.files}))
def test_pairwise_sum_is_numpys(oracle, n):
    a = PW[f"pw/{n}/a"]
    assert oracle.pairwise_sum(a) == float(PW[f"pw/{n}/sum"])


def test_near_tie_classifier(oracle):
    # two centroids equidistant from v: any disagreement is a near-tie
    X = np.array([[0.5, 0.0]], np.float32)
    CB = np.array([[[0.0, 0.0], [1.0, 0.0]]], np.float32)
    n, near, fail, _ = oracle.classify_mismatches(X, CB, np.array([[0]]), np.array([[1]]))
    assert (n, near, fail) == (1, 1, 0)
    X = np.array([[0.1, 0.0]], np.float32)
    n, near, fail, _ = oracle.classify_mismatches(X, CB, np.array([[0]]), np.array([[1]]))
    assert (n, near, fail) == (1, 0, 1)
