"""CPU checks of bench.py's contract pieces that need no GPU: the reference
arm (the oracle on the host cores) prints one JSON line with the required
keys, and the batch workload table names BASELINE's configs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-queries", "4"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["metric"] == "EAT queries/s" and d["higher_is_better"] is True


def test_batch_workloads_table():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.BATCH_WORKLOADS["city_batch"][0] == "city"
    assert bench.BATCH_WORKLOADS["city_batch"][1] == (1000, 10)  # the one 10k batch of BASELINE configs[2]
    assert set(bench.SINGLE_WORKLOADS) == {"city_single", "metro_single", "country_part"}
