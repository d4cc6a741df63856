"""bench.py's JSON line on the GPU (the driver's contract): one line with
the metric / value / e2e / roofline / cpu_baseline / gpu_launches / clocks
keys, launches counted for every timed step, the roofline computed from the
fused kernel's own CUDA-event time, and --gpus N failing loudly on a box
with fewer GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    return subprocess.run([sys.executable, "bench.py", *args], capture_output=True, text=True, timeout=timeout,
                          cwd=ROOT)


def test_default_line_keys():
    r = _run("--steps", "20", "--warmup", "5", "--no-extras", "--cpu-budget-s", "2")
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 5 and d["dtype"] == "f64"
    assert d["config"]["W"] == 1024 and d["config"]["channels"] == 72
    assert d["gpu_launches"] >= 20
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["launches_timed"] == 20 and 0.3 < rf["frac"] < 1.0
    assert abs(rf["achieved"] - rf["bytes_per_launch"] / (rf["avg_kernel_ms"] / 1e3) / 1e9) < 1e-6 * rf["achieved"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["cpu_baseline"] is None or d["cpu_baseline"]["kind"] == "reference"


def test_more_gpus_than_present_fails_loudly():
    import torch
    n = torch.cuda.device_count()
    r = _run("--gpus", str(n + 1), "--steps", "3", timeout=300)
    assert r.returncode != 0
    assert "CUDA device" in (r.stdout + r.stderr)
