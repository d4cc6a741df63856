"""Wire formats on the drop-in boundary: CARMEN log replay
(carmen_log.cpp:9-69) and the scan CSV (observation.cpp:172-208), as
implemented in include/gridloc_b200.hpp, checked against the reference's own
parsers by oracle/ref/dropin_parity.cpp --io-only (host code only: runs on
the CPU). Edge cases follow the reference's test_observation.cpp:360-410 plus
the record grammar's drop rules (no beams, truncated records, other sensors,
non-numeric fields, malformed CSV lines)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_parity")


def test_wire_formats_match_reference(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_parity not built (reference sources absent at build time)")
    env = dict(os.environ, TMPDIR=str(tmp_path))
    r = subprocess.run([BIN, "--io-only"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert lines[-1]["dropin_parity"] == "ok"
    carmen = [x["carmen"] for x in lines if "carmen" in x]
    assert [c["events"] for c in carmen] == [5, 5, 400]
    assert [c["scans"] for c in carmen] == [2, 2, 134]
    assert any("scan_csv" in x and x["scan_csv"]["scans"] == 50 for x in lines)
