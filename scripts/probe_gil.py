"""Where does lloyd_iterate_batched hold the GIL?  A ticker thread increments a counter in pure Python; each
phase of the call reports how many ticks happened during it (few ticks over a long phase = GIL held)."""
import sys, os, time, threading
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C, _native as N
from paper_2605_25521_b200._device import ptr, stream_ptr
dev = torch.device("cuda", 0)
cfg = C.CONFIGS["c2"]
S = C.training_sample(cfg, dev); Ssm = C.subspace_major(S, cfg.m).contiguous(); init = C.lloyd_init(cfg, Ssm)
tc = P.TrainConfig(k=cfg.k, max_iters=cfg.iters, tol=0.0)
P.lloyd_iterate_batched(Ssm, init, tc, return_assignments=False); torch.cuda.synchronize()
ticks = [0]; stop = [False]
def ticker():
    while not stop[0]:
        ticks[0] += 1
        time.sleep(0.0002)
th = threading.Thread(target=ticker, daemon=True); th.start()
def phase(label, fn):
    a, t0 = ticks[0], time.perf_counter(); r = fn(); dt = time.perf_counter() - t0
    print(f"{label:28s} {1e3*dt:7.2f} ms, {ticks[0]-a:4d} ticks (free GIL would give ~{int(dt/0.00026)})"); return r
t = torch
m, n, sub = Ssm.shape; k = cfg.k
Cn = np.array(init if isinstance(init, np.ndarray) else init.cpu().numpy(), dtype=np.float64, copy=True, order="C")
Cd = phase("to_device(C)", lambda: t.from_numpy(Cn).to(dev))
ws = phase("zeros(ws)", lambda: t.zeros(N.load().cspq_lloyd_workspace_bytes(n, m, sub, k), dtype=t.uint8, device=dev))
C32 = t.empty((m, k, sub), dtype=t.float32, device=dev); asg = t.empty((m, n), dtype=t.int32, device=dev)
objs = t.zeros((m, tc.max_iters + 1), dtype=t.float64, device=dev); iters = t.zeros((m,), dtype=t.int32, device=dev)
phase("N.call(cspq_lloyd_train)", lambda: N.call("cspq_lloyd_train", ptr(Ssm), 0, n, m, sub, k, ptr(Cd), tc.max_iters, 0.0, ptr(C32), ptr(asg), ptr(objs), ptr(iters), ptr(ws), stream_ptr(dev)))
phase("C32.cpu()", lambda: C32.cpu())
phase("stream.synchronize()", lambda: t.cuda.current_stream(dev).synchronize())
stop[0] = True
