"""Run on the GPU box: dump full-size training-sample subspaces of configs
c2..c5 (the GPU-generated seeded samples bench.py trains on) so that
tests/golden/make_golden.py can run the reference's own lloyd_iterate on them
here.  Output: gpurun_out/train_samples.npz (points f32, init f64, sha256 of
the subspace points and of the whole sample)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25521_b200 import configs as C  # noqa: E402

PICK = {"c2": (0, 77), "c3": (0, 50), "c4": (17,), "c5": (0, 133)}

dev = torch.device("cuda", 0)
out = {}
for name, js in PICK.items():
    cfg = C.CONFIGS[name]
    S = C.training_sample(cfg, dev)
    Ssm = C.subspace_major(S, cfg.m)
    init = C.lloyd_init(cfg, Ssm)
    out[f"{name}/sample_sha256"] = np.frombuffer(hashlib.sha256(S.cpu().numpy().tobytes()).digest(), np.uint8)
    for j in js:
        p = Ssm[j].cpu().numpy()
        out[f"{name}/{j}/points"] = p
        out[f"{name}/{j}/init"] = init[j]
        out[f"{name}/{j}/points_sha256"] = np.frombuffer(hashlib.sha256(p.tobytes()).digest(), np.uint8)
    print(name, S.shape, js, flush=True)
    del S, Ssm
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/train_samples.npz", **out)
