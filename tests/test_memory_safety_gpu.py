"""Memory-safety and determinism checks of the hot kernels, standing in for
compute-sanitizer (closed on this GPU pool: "runs under it have left GPUs
needing a reset"; profiles/r2_sanitizer.md):

  * out-of-bounds writes (memcheck): every output lives inside a larger
    buffer whose guard bands carry a byte pattern; the pattern must survive
    encode (tcgen05 fix-up and mark modes, guarded / exact SIMT), Lloyd
    training, k-means++ and the host pipeline, on ragged shapes;
  * reads of uninitialised memory (initcheck): outputs pre-filled with
    garbage give the same bits as outputs pre-filled with zeros;
  * races (racecheck / synccheck): repeated runs, including concurrent
    streams, give identical bits.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes of guard band on each side
PAT = 0xA5


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2605_25521_b200 as P
    from paper_2605_25521_b200 import _native as N
    return torch, P, N, torch.device("cuda", 0)


def guarded(torch, dev, nbytes, fill=PAT):
    """A uint8 device buffer of nbytes with guard bands of PAT on both sides; returns (whole, view)."""
    whole = torch.full((nbytes + 2 * GUARD,), fill, dtype=torch.uint8, device=dev)
    whole[:GUARD] = PAT
    whole[GUARD + nbytes:] = PAT
    return whole, whole[GUARD:GUARD + nbytes]


def bands_intact(whole, nbytes):
    h = whole.cpu().numpy()
    return bool((h[:GUARD] == PAT).all() and (h[GUARD + nbytes:] == PAT).all())


def _codebooks(P, m, sub, seed=0, scale=0.3):
    rng = np.random.default_rng(seed)
    rm = (rng.standard_normal((m, 256, sub)) * scale).astype(np.float32)
    return P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])


@pytest.mark.parametrize("n", [1, 5, 127, 128, 129, 1031, 4099])
@pytest.mark.parametrize("mode", ["tensor", "guarded", "exact"])
@pytest.mark.parametrize("shape", [(96, 8, "f32"), (32, 4, "u8"), (16, 8, "f32")])
def test_encode_guard_bands_and_garbage_outputs(env, oracle, n, mode, shape):
    torch, P, N, dev = env
    m, sub, dt = shape
    cs = _codebooks(P, m, sub, scale=30.0 if dt == "u8" else 0.3)
    rng = np.random.default_rng(n)
    if dt == "u8":
        Xh = rng.integers(0, 256, (n, m * sub), dtype=np.uint8)
    else:
        Xh = rng.standard_normal((n, m * sub)).astype(np.float32)
    X = torch.from_numpy(Xh).to(dev)
    want = oracle.encode(Xh, cs.rowmajor, cs.biases, oracle.VARIANT_REFORM)
    outs = []
    for fill in (0x00, 0xFF, 0x5A):
        whole, view = guarded(torch, dev, n * m, fill)
        out = view.view(n, m)
        P.encode_dataset_device(X, cs, P.ExecutionPlan(mode=mode), out=out)
        torch.cuda.synchronize()
        assert bands_intact(whole, n * m), f"encode {mode} wrote outside its {n}x{m} output"
        outs.append(out.cpu().numpy())
    for o in outs:
        assert o.tobytes() == want.tobytes()


def test_encode_tc_best_scores_guard_bands(env):
    torch, P, N, dev = env
    n, m, sub = 1031, 96, 8
    cs = _codebooks(P, m, sub)
    X = torch.randn(n, m * sub, device=dev)
    whole, view = guarded(torch, dev, n * m * 4)
    best = view.view(torch.float32).view(n, m)
    P.encode_dataset_device(X, cs, P.ExecutionPlan(mode="tensor"), best=best)
    torch.cuda.synchronize()
    assert bands_intact(whole, n * m * 4)


def test_lloyd_train_guard_bands_and_garbage_outputs(env, oracle):
    """cspq_lloyd_train through the C ABI: workspace, centroids, assignments and objectives in
    guarded buffers (the workspace zeroed as the ABI requires; outputs pre-filled with garbage)."""
    torch, P, N, dev = env
    rng = np.random.default_rng(7)
    m, n, sub, k, iters = 3, 5003, 8, 256, 6
    cen = rng.uniform(-3, 3, (m, 40, sub))
    pts = np.stack([cen[j][rng.integers(0, 40, n)] + rng.normal(0, 0.4, (n, sub)) for j in range(m)]).astype(np.float32)
    init = pts[:, :k].astype(np.float64).copy()
    init[:, 9] = init[:, 8]  # a duplicate -> an empty cluster -> the repair kernel runs
    Pd = torch.from_numpy(pts).to(dev)
    p = lambda t: t.data_ptr()
    wsb = N.load().cspq_lloyd_workspace_bytes(n, m, sub, k)
    res = []
    for fill in (0x00, 0xFF):
        ws_w, ws = guarded(torch, dev, wsb, 0)
        C64 = torch.from_numpy(init).to(dev)
        c32_w, c32 = guarded(torch, dev, m * k * sub * 4, fill)
        asg_w, asg = guarded(torch, dev, m * n * 4, fill)
        obj_w, obj = guarded(torch, dev, m * (iters + 1) * 8, fill)
        it_w, it = guarded(torch, dev, m * 4, fill)
        N.call("cspq_lloyd_train", p(Pd), 0, n, m, sub, k, p(C64), iters, 0.0, p(c32), p(asg), p(obj), p(it), p(ws),
               torch.cuda.current_stream(dev).cuda_stream)
        torch.cuda.synchronize()
        for w, nb in ((ws_w, wsb), (c32_w, m * k * sub * 4), (asg_w, m * n * 4), (obj_w, m * (iters + 1) * 8),
                      (it_w, m * 4)):
            assert bands_intact(w, nb)
        its = it.view(torch.int32).cpu().numpy()
        objs = obj.view(torch.float64).view(m, iters + 1).cpu().numpy()
        res.append((c32.cpu().numpy().tobytes(), asg.cpu().numpy().tobytes(), its.tobytes(),
                    [objs[j, :its[j] + 1].tobytes() for j in range(m)]))
    assert res[0] == res[1]
    o = oracle.lloyd(pts[1].astype(np.float64), init[1], iters, 0.0)
    assert res[0][0][k * sub * 4:2 * k * sub * 4] == o["centroids"].tobytes()


def test_kmeanspp_guard_bands(env):
    torch, P, N, dev = env
    rng = np.random.default_rng(3)
    m, n, sub, k = 2, 3001, 4, 64
    pts = rng.standard_normal((m, n, sub)).astype(np.float32)
    Pd = torch.from_numpy(pts).to(dev)
    first = torch.tensor([5, 17], dtype=torch.int64, device=dev)
    u = torch.from_numpy(rng.random((m, k))).to(dev)
    p = lambda t: t.data_ptr()
    wsb = N.load().cspq_lloyd_workspace_bytes(n, m, sub, k)
    outs = []
    for fill in (0x00, 0xFF):
        ws_w, ws = guarded(torch, dev, wsb, 0)
        c_w, c = guarded(torch, dev, m * k * sub * 8, fill)
        s_w, s = guarded(torch, dev, m * 4, 0)
        N.call("cspq_kmeanspp", p(Pd), 0, n, m, sub, k, p(first), p(u), p(c), p(s), p(ws),
               torch.cuda.current_stream(dev).cuda_stream)
        torch.cuda.synchronize()
        assert bands_intact(ws_w, wsb) and bands_intact(c_w, m * k * sub * 8) and bands_intact(s_w, m * 4)
        outs.append(c.cpu().numpy().tobytes())
    assert outs[0] == outs[1]


def test_repeated_and_concurrent_runs_are_bitwise_identical(env):
    """Racecheck stand-in: the warp-specialised tcgen05 pipeline (mbarrier ring, TMEM double
    buffer), the SIMT kernels and the Lloyd loop give the same bits run after run, also when
    two streams run them concurrently."""
    torch, P, N, dev = env
    n, m, sub = 300_000, 96, 8
    cs = _codebooks(P, m, sub)
    X = torch.randn(n, m * sub, device=dev)
    X /= X.norm(dim=1, keepdim=True)
    ref = {mode: P.encode_dataset_device(X, cs, P.ExecutionPlan(mode=mode)).cpu().numpy()
           for mode in ("tensor", "guarded")}
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for _ in range(3):
        outs = {}
        for mode, s in (("tensor", s1), ("guarded", s2)):
            with torch.cuda.stream(s):
                outs[mode] = P.encode_dataset_device(X, cs, P.ExecutionPlan(mode=mode))
        torch.cuda.synchronize()
        for mode in outs:
            assert outs[mode].cpu().numpy().tobytes() == ref[mode].tobytes()
    assert ref["tensor"].tobytes() == ref["guarded"].tobytes()
    rng = np.random.default_rng(1)
    pts = rng.standard_normal((4, 20_000, 8)).astype(np.float32)
    init = pts[:, :256].astype(np.float64)
    cfg = P.TrainConfig(k=256, max_iters=8, tol=0.0)
    first = P.lloyd_iterate_batched(pts, init, cfg)
    for _ in range(2):
        again = P.lloyd_iterate_batched(pts, init, cfg)
        for a, b in zip(first, again):
            assert a.centroids.tobytes() == b.centroids.tobytes() and a.objectives == b.objectives
            assert np.array_equal(a.assignments, b.assignments)


def test_host_pipeline_guard_bands(env):
    """cspq_encode_host writes exactly n * m codes into the caller's host buffer (pinned and
    pageable, with and without cudaHostRegister), on ragged batch splits."""
    import os
    torch, P, N, dev = env
    n, m, sub = 10_007, 16, 8
    cs = _codebooks(P, m, sub)
    rng = np.random.default_rng(2)
    X = rng.standard_normal((n, m * sub)).astype(np.float32)
    want = P.encode_dataset_device(torch.from_numpy(X).to(dev), cs).cpu().numpy()
    for reg in ("0", "1"):
        os.environ["CSPQ_HOST_REGISTER"] = reg
        try:
            for pinned in (False, True):
                buf = (P.pinned_empty((n * m + 2 * GUARD,), np.uint8) if pinned
                       else np.empty(n * m + 2 * GUARD, np.uint8))
                buf[:] = PAT
                out = buf[GUARD:GUARD + n * m].reshape(n, m)
                P.encode_dataset_host(X, cs, P.ExecutionPlan(batch_rows=999, streams=3), out=out)
                assert (buf[:GUARD] == PAT).all() and (buf[GUARD + n * m:] == PAT).all()
                assert out.tobytes() == want.tobytes()
        finally:
            os.environ.pop("CSPQ_HOST_REGISTER", None)


def test_host_api_rejects_bad_out_and_batch_ms(env):
    torch, P, N, dev = env
    cs = _codebooks(P, 4, 8)
    X = np.zeros((100, 32), np.float32)
    for bad in (np.empty((100, 4), np.uint16), np.empty((100, 5), np.uint8), np.empty((4, 100), np.uint8).T,
                np.empty((99, 4), np.uint8)):
        with pytest.raises(P.ConfigError):
            P.encode_dataset_host(X, cs, out=bad)
    with pytest.raises(P.ConfigError):
        P.encode_dataset_host(X, cs, P.ExecutionPlan(batch_rows=10), batch_ms=np.zeros(9, np.float64))
    with pytest.raises(P.ConfigError):
        P.encode_dataset_host(X, cs, P.ExecutionPlan(batch_rows=10), batch_ms=np.zeros(10, np.float32))


def test_uint8_misaligned_views_fall_back_instead_of_faulting(env, oracle):
    """a uint8 view at an odd offset must not reach the tcgen05 kernel's sub-byte
    cp.async (the C ABI rejects it with CSPQ_E_CONFIG; the Python path uses the SIMT kernel)."""
    torch, P, N, dev = env
    m, sub = 32, 4
    cs = _codebooks(P, m, sub, scale=30.0)
    rng = np.random.default_rng(9)
    big = rng.integers(0, 256, (777, m * sub + 3), dtype=np.uint8)
    Xd = torch.from_numpy(big).to(dev)[:, 1:1 + m * sub]  # odd base offset and odd row stride
    want = oracle.encode(np.ascontiguousarray(big[:, 1:1 + m * sub]), cs.rowmajor, cs.biases, oracle.VARIANT_REFORM)
    got = P.encode_dataset_device(Xd, cs).cpu().numpy()
    assert got.tobytes() == want.tobytes()
    rm, bs, guard, _, _ = cs.on_device(dev)
    img = cs.tc_image(dev)
    codes = torch.empty((777, m), dtype=torch.uint8, device=dev)
    rc = N.load().cspq_encode_tc(ctypes.c_void_p(Xd.data_ptr()), N.IN_U8, 777, m * sub, Xd.stride(0),
                                 ctypes.c_void_p(rm.data_ptr()), ctypes.c_void_p(bs.data_ptr()),
                                 ctypes.c_void_p(guard.data_ptr()), ctypes.c_void_p(img.data_ptr()), m, 256, sub,
                                 ctypes.c_void_p(codes.data_ptr()), m, None,
                                 ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    assert rc == N.CSPQ_E_CONFIG
    torch.cuda.synchronize()
