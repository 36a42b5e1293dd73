import sys, os, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2605_25521_b200 as P
from paper_2605_25521_b200 import configs as C
dev = torch.device("cuda", 0)
cfg = C.CONFIGS["c3"]; n = 4_000_000
X = C.generate(cfg, 0, n, dev)
rng = np.random.default_rng(0)
rows = X[torch.from_numpy(rng.choice(n, cfg.k, replace=False)).to(dev)].float().cpu().numpy()
rm = np.ascontiguousarray(rows.reshape(cfg.k, cfg.m, cfg.sub).transpose(1, 0, 2))
cs = P.CodebookSet.from_codebooks([P.Codebook.from_rowmajor(j, rm[j]) for j in range(cfg.m)])
plan = P.ExecutionPlan(mode="tensor")
out = P.encode_dataset_device(X, cs, plan); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): P.encode_dataset_device(X, cs, plan, out=out)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("CSPQ_TC_PROBE", "0"), e0.elapsed_time(e1) / 3, "ms")
'''
for pr in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "8", "1", "4", "12", "2"]):
    env = dict(os.environ, CSPQ_TC_PROBE=pr)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(r.stdout.strip(), r.stderr.strip()[-200:] if r.returncode else "", flush=True)
