"""Timeline of chunked H2D uploads (side stream, window 2) with and without a Lloyd training running beside them."""
import sys, os, time, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
cfg = C.CONFIGS["c2"]
S = C.training_sample(cfg, dev); Ssm = C.subspace_major(S, cfg.m); init = C.lloyd_init(cfg, Ssm)
tc = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
Xh = P.pinned_empty((1_000_000, cfg.d), np.float32); Xh[:] = 0.5
src = torch.from_numpy(Xh); Xd = torch.empty(src.shape, dtype=src.dtype, device=dev)
side = torch.cuda.Stream(dev); rows_per = (64 << 20) // Xh.strides[0]
def feed(stamps, t0):
    with torch.cuda.device(dev), torch.cuda.stream(side):
        evs = []
        for r0 in range(0, src.shape[0], rows_per):
            if len(evs) >= 2:
                evs.pop(0).synchronize()
            stamps.append(time.perf_counter() - t0)
            Xd[r0:r0 + rows_per].copy_(src[r0:r0 + rows_per], non_blocking=True)
            e = torch.cuda.Event(); e.record(side); evs.append(e)
        side.synchronize(); stamps.append(time.perf_counter() - t0)
def train_dev(): return P.lloyd_iterate_batched(Ssm, init, tc, return_assignments=False)   # device-resident sample: no H2D of its own
train_dev(); torch.cuda.synchronize()
for label, fn in (("upload alone", None), ("upload || training (device-resident sample)", train_dev)):
    st = []; t0 = time.perf_counter()
    th = threading.Thread(target=feed, args=(st, t0)); th.start()
    if fn:
        fn(); tr = time.perf_counter() - t0
    th.join(); torch.cuda.synchronize()
    ms = [round(1e3 * v, 1) for v in st]
    print(label, "total", ms[-1], "ms", ("train returned at %.1f" % (1e3 * tr)) if fn else "", "chunk issue times:", ms[::6], "first 8:", ms[:8])
A = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
def gpu_busy():
    for _ in range(40): (A @ A)
    torch.cuda.synchronize()
def cpu_busy():
    x = 0
    t = time.perf_counter()
    while time.perf_counter() - t < 0.03: x += 1
gpu_busy()
for label, fn in (("upload || matmuls (torch, GIL released in synchronize)", gpu_busy), ("upload || python busy loop (GIL held, no GPU)", cpu_busy)):
    st = []; t0 = time.perf_counter()
    th = threading.Thread(target=feed, args=(st, t0)); th.start()
    fn(); tr = time.perf_counter() - t0
    th.join(); torch.cuda.synchronize()
    ms = [round(1e3 * v, 1) for v in st]
    print(label, "total", ms[-1], "ms", "fn returned at %.1f" % (1e3 * tr), "chunk issue times:", ms[::6], "first 8:", ms[:8])
small = torch.zeros(1024, device=dev)
def gpu_busy_then_d2h():
    for _ in range(40): (A @ A)
    return small.cpu()
def gpu_busy_sync_then_d2h():
    for _ in range(40): (A @ A)
    torch.cuda.current_stream(dev).synchronize()
    return small.cpu()
for label, fn in (("upload || matmuls then .cpu() queued behind them", gpu_busy_then_d2h), ("upload || matmuls, stream sync, then .cpu()", gpu_busy_sync_then_d2h)):
    st = []; t0 = time.perf_counter()
    th = threading.Thread(target=feed, args=(st, t0)); th.start()
    fn(); tr = time.perf_counter() - t0
    th.join(); torch.cuda.synchronize()
    ms = [round(1e3 * v, 1) for v in st]
    print(label, "total", ms[-1], "ms", "fn returned at %.1f" % (1e3 * tr), "first 8:", ms[:8])
