"""The driver's bench.py contract, checked on CPU through the reference arm
(the C oracle; no GPU): one JSON line with the required keys."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["metric"] == "PQ-encoded vectors/sec" and j["unit"] == "vectors/s"
    assert j["value"] > 0 and j["steps"] == 1 and j["higher_is_better"] is True
    assert j["cpu_baseline"]["kind"] in ("reference", "port") and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["value"] == j["value"] and j["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in j["config"]


def test_strong_scaling_shards_the_config_rows():
    """c2-c5 shard the config's N across ranks (c3 at 8 GPUs: 1,250,000 rows each, global 10M);
    c1 runs replicas."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2605_25521_b200 import configs as C
    args = bench.parse([])
    c3 = C.CONFIGS["c3"]
    spans = [bench.rows_of(args, c3, 8, r) for r in range(8)]
    assert all(e - b == 1_250_000 and g == 10_000_000 for b, e, g in spans)
    assert spans[0][0] == 0 and spans[-1][1] == 10_000_000
    assert "1,250,000 rows/GPU, global 10,000,000" in bench.workload_desc(c3, 1_250_000, 10_000_000, 8, "strong")
    c4 = C.CONFIGS["c4"]
    assert sum(e - b for b, e, _ in (bench.rows_of(args, c4, 8, r) for r in range(8))) == 200_000_000
    c1 = C.CONFIGS["c1"]
    assert bench.scaling_of(args, c1) == "weak" and bench.rows_of(args, c1, 2, 1) == (100_000, 200_000, 200_000)
    assert args.reduce == "allgather" and args.train == "auto"
