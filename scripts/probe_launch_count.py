"""Probe: does torch.profiler (CUPTI) see this repo's kernel launches on repeated sessions?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
from torch.profiler import ProfilerActivity, profile
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
rm = (rng.standard_normal((96, 256, 8)) * 0.1).astype(np.float32)
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(96)])
X = torch.randn(100000, 768, device=dev)
out = P.encode_dataset_device(X, cs)
for it in range(4):
    with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
        P.encode_dataset_device(X, cs, out=out)
        torch.cuda.synchronize()
    evs = list(prof.events())
    names = [(str(getattr(e, "device_type", None)), (e.name or "")[:80]) for e in evs]
    print(it, len(evs), names[:6], flush=True)
    ka = prof.key_averages()
    print("  ka", [(k.key[:60], k.count) for k in ka][:6], flush=True)
