"""CPU-only tests: the C-ABI library loads and exports every symbol the
header declares, the host-side API mirrors the reference's validation and
data model (pkg/tests/test_core.py, test_bulk.py plan/codebook tests), and
the product path refuses to run without CUDA (no silent CPU fallback)."""

import numpy as np
import pytest

import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import _native as N


def test_library_exports_every_header_symbol():
    L = N.load()
    declared = N.header_symbols()
    assert set(declared) == set(N.exported_symbols())
    for name in declared:
        assert hasattr(L, name), name
    assert L.cspq_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_cuda(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    cb = P.Codebook.from_rowmajor(0, np.eye(4, dtype=np.float32))
    with pytest.raises(P.NativeUnavailable):
        P.encode_ref([1, 0, 0, 0], cb)
    with pytest.raises(P.NativeUnavailable):
        P.encode_dataset(np.zeros((3, 4), np.float32), [cb])
    with pytest.raises(P.NativeUnavailable):
        P.lloyd_iterate(np.zeros((4, 1)), np.zeros((2, 1)), P.TrainConfig(k=2))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(N.NativeUnavailable):
        N.load()


def test_c_abi_validation_errors_map_to_reference_exceptions():
    # argument checks run before any device work, so they work without a GPU
    with pytest.raises(P.ConfigError, match="dimensionality"):
        N.call("cspq_encode", None, 0, 5, 10, 10, None, None, None, 2, 256, 4, None, 2, 1, 0, None)
    with pytest.raises(P.ConfigError, match="k must be"):
        N.call("cspq_encode", None, 0, 5, 8, 8, None, None, None, 2, 0, 4, None, 2, 1, 0, None)
    with pytest.raises(P.ConfigError, match="bad variant"):
        N.call("cspq_encode", None, 0, 5, 8, 8, None, None, None, 2, 256, 4, None, 2, 7, 0, None)
    # empty input is a successful no-op
    assert N.call("cspq_encode", None, 0, 0, 8, 8, None, None, None, 2, 256, 4, None, 2, 1, 0, None) == 0
    with pytest.raises(P.TrainingError):
        N.call("cspq_lloyd_train", 1, 0, 10, 1, 4, 16, 1, 0, 0.0, 1, 1, 1, 1, 1, None)


class TestPlanAndCodebooks:
    def test_plan_validation(self):
        with pytest.raises(P.ConfigError):
            P.ExecutionPlan(order="diagonal")
        with pytest.raises(P.ConfigError):
            P.ExecutionPlan(workers=0)
        with pytest.raises(P.ConfigError):
            P.ExecutionPlan(block_size=0)
        with pytest.raises(P.ConfigError):
            P.ExecutionPlan(w=0)
        with pytest.raises(P.ConfigError):
            P.ExecutionPlan(mode="fast")
        assert P.ExecutionPlan().resolved_w() in (4, 8, 16)
        # ~256 MB of rows, not derived from block_size (a 1M-row block must not size a 9 GB ring)
        assert P.ExecutionPlan(block_size=1_000_000).resolved_batch_rows(3072) == (256 << 20) // 3072
        assert P.ExecutionPlan().resolved_batch_rows(128) == 1 << 20
        assert P.ExecutionPlan().resolved_batch_rows(1 << 20) == 1 << 14
        assert P.ExecutionPlan(batch_rows=4096).resolved_batch_rows() == 4096

    def test_codebook_set(self):
        rng = np.random.default_rng(31)
        cbs = [P.Codebook.from_rowmajor(j, rng.standard_normal((24, 4)).astype(np.float32)) for j in range(3)]
        cs = P.CodebookSet.from_codebooks(cbs)
        assert (cs.m, cs.k, cs.sub_dim, cs.d) == (3, 24, 4, 12)
        assert np.array_equal(cs[1].centroids_rowmajor, cbs[1].centroids_rowmajor)
        assert np.array_equal(cs[1].biases, cbs[1].biases)
        assert P.CodebookSet.from_codebooks(cs) is cs
        b = P.Codebook.from_rowmajor(1, rng.standard_normal((9, 4)).astype(np.float32))
        with pytest.raises(P.ConfigError):
            P.CodebookSet.from_codebooks([cbs[0], b])
        with pytest.raises(P.ConfigError):
            P.CodebookSet.from_codebooks([])

    def test_working_set(self):
        assert P.estimate_working_set(P.PQParams(d=256, m=16, k=256, w=8), P.ExecutionPlan(w=8)) == 33_792 + 64
        assert P.estimate_working_set(P.PQParams(d=16, m=4, k=16, w=4),
                                      P.ExecutionPlan(w=4, workers=2)) == 576 + 64


class TestCore:
    def test_params(self):
        with pytest.raises(P.ConfigError):
            P.PQParams(d=10, m=3)
        with pytest.raises(P.ConfigError):
            P.PQParams(d=8, m=2, k=0)
        with pytest.raises(P.ConfigError):
            P.PQParams(d=8, m=2, k=70000)
        assert P.PQParams(d=12, m=3).sub_dim == 4

    def test_layouts_and_biases(self):
        rng = np.random.default_rng(2)
        rm = rng.standard_normal((17, 5)).astype(np.float32)
        t = P.transpose_codebook(rm)
        assert t.shape == (5, 17) and np.array_equal(P.transpose_codebook(t), rm)
        ref = (0.5 * (rm.astype(np.float64) ** 2).sum(axis=1)).astype(np.float32)
        assert np.allclose(P.compute_biases(rm), ref, rtol=1e-7, atol=0)
        with pytest.raises(P.FormatError):
            P.transpose_codebook([[1, 2], [3]])
        with pytest.raises(P.DataError):
            P.compute_biases(np.array([[np.nan, 1.0]], np.float32))
        cb = P.Codebook.from_rowmajor(0, rm)
        assert not cb.centroids_rowmajor.flags.writeable
        with pytest.raises(P.DataError):
            P.Codebook.from_rowmajor(0, np.array([[np.inf, 0]], np.float32))

    def test_codes_and_dataset(self):
        with pytest.raises(P.CorruptionError):
            P.PQCodes(codes=np.array([[5]], np.uint8), k=4)
        with pytest.raises(P.ConfigError):
            P.PQCodes(codes=np.array([[1]], np.int32), k=4)
        c = P.PQCodes(codes=np.zeros((3, 2), np.uint16), k=300)
        assert (c.n, c.m) == (3, 2)
        with pytest.raises(P.ConfigError):
            P.VectorDataset(data=np.zeros((3, 2), np.float64))
        with pytest.raises(P.DataError):
            P.VectorDataset(data=np.array([[np.nan]], np.float32))

    def test_partition(self):
        parts = P.partition_vector(np.arange(12, dtype=np.float32), P.PQParams(d=12, m=3))
        assert [p.tolist() for p in parts] == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11]]
        with pytest.raises(P.ConfigError):
            P.partition_vector(np.arange(10, dtype=np.float32), P.PQParams(d=12, m=3))

    def test_train_config(self):
        with pytest.raises(P.TrainingError):
            P.TrainConfig(k=0)
        with pytest.raises(P.TrainingError):
            P.TrainConfig(max_iters=0)
        with pytest.raises(P.TrainingError):
            P.TrainConfig(tol=-1)
        assert P.TrainConfig(k=16).resolved_cap() == 4096
        assert P.TrainConfig(sample_cap=0).resolved_cap() is None


def test_configs_host_definitions():
    from paper_2605_25521_b200 import configs as C
    c3 = C.CONFIGS["c3"]
    assert (c3.n, c3.d, c3.m, c3.sub, c3.k) == (10_000_000, 768, 96, 8, 256)
    assert C.CONFIGS["c4"].sub == 4 and C.CONFIGS["c4"].elem_bytes == 1
    assert c3.flops_per_vec() == 2 * 256 * 768 and c3.bytes_per_vec() == 768 * 4 + 96
    idx = C.sample_indices(c3.scaled(n=10_000, n_train=500))
    assert idx.shape == (500,) and np.all(np.diff(idx) > 0)
    assert np.array_equal(idx, C.sample_indices(c3.scaled(n=10_000, n_train=500)))


def test_encode_dataset_device_rejects_host_tensors_and_bad_outputs():
    """Argument checks that run before any CUDA call (no GPU needed)."""
    import torch
    import paper_2605_25521_b200 as P
    rm = np.random.default_rng(0).standard_normal((2, 256, 4)).astype(np.float32)
    cbs = [P.Codebook.from_rowmajor(j, rm[j]) for j in range(2)]
    with pytest.raises(P.ConfigError, match="CUDA tensor"):
        P.encode_dataset_device(torch.zeros((4, 8)), cbs)
    with pytest.raises(P.ConfigError, match="CUDA tensor"):
        P.encode_dataset_device(np.zeros((4, 8), np.float32), cbs)


def test_execution_plan_devices_validation():
    assert P.ExecutionPlan(devices=[0, 1]).devices == (0, 1)
    assert P.ExecutionPlan(devices=np.array([2, 3])).devices == (2, 3)
    for bad in ([], [-1], [0.5], ["0"]):
        with pytest.raises(P.ConfigError, match="devices"):
            P.ExecutionPlan(devices=bad)


def test_tensor_kernel_subspace_limit_query():
    L = N.load()
    for sub in (4, 8):
        for dt in (N.IN_F32, N.IN_U8):
            assert L.cspq_encode_tc_max_subspaces(sub, dt) >= 256  # every configuration (m <= 192) fits
    assert L.cspq_encode_tc_max_subspaces(16, N.IN_F32) == 0


def test_codebookset_from_rowmajor_batch_equals_per_subspace_construction():
    """CodebookSet.from_rowmajor_batch builds the arrays of from_codebooks([Codebook.from_rowmajor ...])
    bit for bit (the biases are part of the encode contract), and rejects what they reject."""
    import numpy as np
    import pytest
    import paper_2605_25521_b200 as P
    rng = np.random.default_rng(5)
    for m, k, sub in [(1, 1, 1), (3, 7, 3), (16, 256, 8), (5, 256, 4), (2, 300, 16), (4, 33, 5)]:
        C = (rng.standard_normal((m, k, sub)) * rng.choice([1e-3, 1.0, 300.0])).astype(np.float32)
        a = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, C[j]) for j in range(m)])
        b = P.CodebookSet.from_rowmajor_batch(C)
        for x, y in ((a.rowmajor, b.rowmajor), (a.transposed, b.transposed), (a.biases, b.biases)):
            assert x.dtype == y.dtype and x.shape == y.shape and x.tobytes() == y.tobytes()
            assert not y.flags.writeable
    bad = np.zeros((3, 4, 2), np.float32)
    bad[1, 2, 0] = np.nan
    with pytest.raises(P.DataError, match="subspace 1"):
        P.CodebookSet.from_rowmajor_batch(bad)
    with pytest.raises(P.ConfigError):
        P.CodebookSet.from_rowmajor_batch(np.zeros((4, 2), np.float32))
