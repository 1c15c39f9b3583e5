"""The driver's bench contract on a small workload (config B size): one JSON line
with the required keys, a roofline and CPU baseline, and a converged
time-to-solution leg."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_json_line_small():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
         "--target-nodes", "100000"],
        capture_output=True, text=True, timeout=900, check=True)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "pcg"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["steps"] == 3
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in d["roofline"], key
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["pcg"]["converged"] and d["pcg"]["true_relres"] < 1.01e-6
    assert d["cpu_baseline"]["value"] > 0
    assert d["pcg_flexible"]["converged"]
    assert d["time_to_solution_small"]["A"]["converged"]
