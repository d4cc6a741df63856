"""Drop-in check through the C++ API (include/gridloc_b200.hpp): the same
driver code against the reference gridloc:: and against gridloc_b200::,
linked side by side (oracle/ref/dropin_parity.cpp, built by oracle/Makefile
where the reference sources exist; the prebuilt binary travels to the GPU
box). Covers step bit-exactness for four kernel sets, argmax / belief_map /
dither, and two full Localizer runs with LIDAR observations."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_parity")

pytestmark = pytest.mark.gpu


def test_cpp_dropin_parity():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_parity not built (reference sources absent at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    last = json.loads(r.stdout.strip().splitlines()[-1])
    assert last["dropin_parity"] == "ok"
