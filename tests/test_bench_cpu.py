"""bench.py's reference arm runs on the host alone (SURVEY.md §8d CPU baseline):
one JSON line with the contract's keys, on a small workload."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "1", "--target-nodes", "5000", "--subdomain-size", "1000"],
        capture_output=True, text=True, timeout=600, check=True)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    # the reference process maps none of this repository's native libraries
    assert d["native_libs_mapped"] == []
    assert d["pcg_config_a"]["converged"] and d["pcg_config_a"]["iterations"] > 0
    assert "N=4762" in d["config"]["workload"]
