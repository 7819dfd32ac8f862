"""bench.py's output contract, CPU only: the reference arm (--impl reference) runs the
reference's own CPU ChebyPower (oracle/_ref) on config 1 and must print exactly ONE JSON
line on stdout with the driver's keys, without loading the product library."""
import json
import os
import subprocess
import sys

import pytest

from oracle import Ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not Ref.available(), reason="reference library not built")
def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                        "--warmup", "1", "--cpu-budget", "2"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, r.stdout[:2000]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GTEPS" and d["value"] > 0
    assert d["config"]["workload"] and d["config"]["n"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["whole_queries"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["product_library_loaded"] is False  # the reference arm maps only oracle/ libraries
