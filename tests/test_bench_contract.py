"""bench.py --impl reference: the reference arm's JSON line (runs on CPU).

The driver computes the our-arm / reference-arm ratio itself, so the reference
line must carry the same metric, unit, direction, dtype and workload config.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                        "--cpu-sample", "200000"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    import bench
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == "records/s" and d["higher_is_better"] is True
    assert d["dtype"] == "int64" and d["value"] > 0
    c = d["config"]
    assert c["workload"] == "C2" and c["algorithm"] == "pre_partitioning"
    assert c["records_per_gpu"] == 100_000_000 and c["budget_groups"] == 125_000
    assert c["records_per_step"] == 200_000
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
