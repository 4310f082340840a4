"""bench.py contract on CPU: the reference arm runs the reference's own
passes side by side on the host cores and prints the same config dict the
b200 arm prints (the driver pairs the two lines by it)."""
import json
import os
import subprocess
import sys
from types import SimpleNamespace

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_workload_config_is_shared():
    a = SimpleNamespace(mesh="genus:8:45", pass_steps=3000)
    c = bench.workload_config(a, 988186, 1)
    assert c["genus"] == 8 and c["vertices"] == 988186 and c["pass_steps"] == 3000
    assert c["parallelism"] == "replicas x1"
    assert bench.workload_config(SimpleNamespace(mesh="gyroid:2:26:0.3:1.0", pass_steps=10), 5, 2)["genus"] is None


def test_reference_concurrency_bounds():
    assert bench.reference_concurrency(1) == 1
    assert 1 <= bench.reference_concurrency(1000) <= (os.cpu_count() or 1)


@pytest.mark.skipif(not os.path.exists(bench.REF_BIN), reason="oracle/_ref not built")
def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                          "--warmup", "1", "--pass-steps", "5", "--mesh", "genus:2:10"],
                         check=True, capture_output=True, text=True, timeout=300)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 3 and line["warmup"] == 1
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"] == bench.workload_config(SimpleNamespace(mesh="genus:2:10", pass_steps=5),
                                                   line["config"]["vertices"], 1)
