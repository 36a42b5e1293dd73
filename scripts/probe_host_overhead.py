"""Host-side cost per encode call: the Python API (encode_dataset_device) and the raw C call."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import _native as N
from paper_2605_25521_b200._device import ptr, stream_ptr
rng = np.random.default_rng(0)
m, sub = 16, 8
rm = rng.standard_normal((m, 256, sub)).astype(np.float32)
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(m)])
X = torch.from_numpy(rng.standard_normal((128, m * sub)).astype(np.float32)).cuda()
out = P.encode_dataset_device(X, cs); torch.cuda.synchronize()
plan = P.ExecutionPlan()
for name, fn in [("encode_dataset_device", lambda: P.encode_dataset_device(X, cs, plan, out=out))]:
    for _ in range(50): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(2000): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(name, f"host {1e6*(t1-t)/2000:.1f} us/call, incl. drain {1e6*(t2-t)/2000:.1f} us/call")
dev = X.device
rm_d, bs, guard, vid = P.bulk._variant_args(cs, plan, True, dev)
img = cs.tc_image(dev)
sp = stream_ptr(dev)
def raw():
    N.call("cspq_encode_tc", ptr(X), N.IN_F32, 128, m * sub, m * sub, ptr(rm_d), ptr(bs), ptr(guard), ptr(img), m, 256, sub, ptr(out), m, None, sp)
for _ in range(50): raw()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(2000): raw()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("raw C call", f"host {1e6*(t1-t)/2000:.1f} us/call, incl. drain {1e6*(t2-t)/2000:.1f} us/call")
