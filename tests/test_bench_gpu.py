"""bench.py contract checks on the GPU (short runs): the default line carries
every key the driver reads (metric, value, unit, n_gpus, steps, warmup,
ms_per_step, higher_is_better, scaling, vs_baseline, dtype, data, config,
clocks, e2e, gpu_launches, roofline, cpu_baseline, maml_c4), the MAML and
reference arms print valid lines, and the peer-memory outer step runs."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, timeout=600):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_default_line_keys():
    d = run("--steps", "20", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "clocks",
              "e2e", "gpu_launches", "roofline", "cpu_baseline", "maml_c4"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] >= 3
    assert d["value"] > 0 and d["gpu_launches"] == 40
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["unit"] == "GB/s"
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["maml_c4"].get("value", 0) > 0, d["maml_c4"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_line():
    d = run("--impl", "reference", "--steps", "2", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("outer", ["adam", "peer"])
def test_maml_line(outer):
    d = run("--workload", "maml", "--tasks", "4", "--steps", "3", "--warmup", "3",
            "--maml-outer", outer)
    assert d["unit"] == "tasks/s" and d["value"] > 0 and d["config"]["tasks"] == 4
