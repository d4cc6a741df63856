"""bench.py's contract pieces that run on CPU: the reference arm never maps
the product library, prints the same config dict as our arm, and carries
the cpu_baseline detail SURVEY §8(d) asks for (lscpu model, median / p99)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_input_generator_does_not_map_the_product():
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "from paper_1910_00572_b200.floorplan import make_floorplan; make_floorplan(64, 64); "
            "print(bench.product_not_mapped())" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.stdout.strip().splitlines()[-1] == "True", out.stderr[-2000:]


def test_reference_arm_line():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "5",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    sys.path.insert(0, ROOT)
    import bench
    assert line["impl"] == "reference"
    assert line["config"] == bench.config_for(bench.CONFIGS["c1"])  # identical to our arm's dict
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["product_library_mapped"] is False
    assert {"median_ms", "p99_ms", "cpu_model", "cores"} <= set(cb)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
