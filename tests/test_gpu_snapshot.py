"""BLF1 belief snapshots (belief_tensor.hpp:144-148, belief_tensor.cpp:
543-587) against the reference's own writer and reader: byte-identical
files for the same belief, identical values and theta_t when reading the
reference's file, and the reference's error cases. The float32 conversion
runs on the device (round-to-nearest, like static_cast<float>)."""
import math
import os

import numpy as np
import pytest

import oracle
import paper_1910_00572_b200 as g
from tests.helpers import make_floorplan

pytestmark = pytest.mark.gpu


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def test_write_matches_reference_bytes(ctx, ref, tmp_path):
    # the reference test's shape (test_belief_engine.cpp:520-537) and a
    # stepped floor-plan belief with a pending rescale-free history
    rng = np.random.default_rng(8)
    cases = [(rng.random((4, 5, 7)), 1.25)]
    occ = make_floorplan(96, 64, seed=5)
    m = g.OccupancyMap(96, 64, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), 72, 0.1, 2 * math.pi / 72)
    act = g.make_activation(m, ks, 72, ctx)
    t = g.init_uniform(m, 72, ctx)
    for u in [(0.1, 0.0, 0.0), (0.05, 0.02, 0.3)]:
        g.step(t, g.OdometryDelta(*u), m, ks, act, ctx)
    cases.append((t.values(), t.theta_t()))
    for i, (vals, th) in enumerate(cases):
        c, h, w = vals.shape
        gt = g.BeliefTensor(w, h, c, 0.1, ctx=ctx)
        gt.set_values(vals)
        gt.set_theta_t(th)
        ours, theirs = str(tmp_path / f"g{i}.blf"), str(tmp_path / f"r{i}.blf")
        g.write_belief_snapshot(gt, ours)
        oracle.ref_write_snapshot(ref, vals, th, theirs)
        assert _bytes(ours) == _bytes(theirs), f"case {i}: BLF1 bytes differ"
        assert len(_bytes(ours)) == 20 + 4 * vals.size


def test_read_matches_reference_reader(ctx, ref, tmp_path):
    vals = np.random.default_rng(3).random((8, 12, 16)) * 1e-3
    p = str(tmp_path / "r.blf")
    oracle.ref_write_snapshot(ref, vals, -2.5, p)
    t = g.read_belief_snapshot(p, 0.25, 0.0, 0.0, ctx=ctx)
    rv, rth = oracle.ref_read_snapshot(ref, p, 0.25)
    assert (t.width(), t.height(), t.channels()) == (16, 12, 8)
    assert t.theta_t() == rth
    assert np.array_equal(t.values().view(np.uint64), rv.view(np.uint64))
    # round trip of the reference test: float32 payload, 1e-6 relative
    assert np.allclose(t.values(), vals, rtol=1e-6, atol=0)


def test_snapshot_errors_match_reference(ctx, tmp_path):
    with pytest.raises(g.GridlocError, match="cannot open snapshot"):
        g.read_belief_snapshot(str(tmp_path / "missing.blf"), 0.1, 0.0, 0.0, ctx=ctx)
    bad = tmp_path / "bad.blf"
    bad.write_bytes(b"BLF2" + bytes(16))
    with pytest.raises(g.GridlocError, match="bad belief snapshot magic"):
        g.read_belief_snapshot(str(bad), 0.1, 0.0, 0.0, ctx=ctx)
    short = tmp_path / "short.blf"
    short.write_bytes(b"BLF1" + np.array([4, 4, 4], np.uint32).tobytes() + np.float32(0).tobytes() + bytes(10))
    with pytest.raises(g.GridlocError, match="truncated belief snapshot"):
        g.read_belief_snapshot(str(short), 0.1, 0.0, 0.0, ctx=ctx)
    t = g.BeliefTensor(4, 4, 4, 0.1, ctx=ctx)
    with pytest.raises(g.GridlocError, match="cannot open for writing"):
        g.write_belief_snapshot(t, str(tmp_path / "no" / "such" / "dir.blf"))
