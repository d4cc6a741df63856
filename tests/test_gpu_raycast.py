"""Device raycast / simulate_scan batches (batch trace
generation) against the UNMODIFIED reference (oracle/_ref):
raycast occupancy_map.cpp:273-332 and simulate_scan simulator.cpp:63-94,
bit-exact ranges and angles, with and without range noise (the reference's
Rng draw order), corner ties (45-degree beams), partial fields of view, and
the reference's errors."""
import math

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from paper_1910_00572_b200.floorplan import Rng
from tests.helpers import make_floorplan, random_map

pytestmark = pytest.mark.gpu


def _ref_scan(ref, rm, pose, beams, fov, max_range, sigma, seed):
    import oracle
    a, r = np.zeros(beams), np.zeros(beams)
    ref.check(ref.lib.ref_simulate_scan(rm.h, pose[0], pose[1], pose[2], beams, fov, max_range, sigma, seed,
                                        oracle._d(a), oracle._d(r)), "scan")
    return a, r


def _free_poses(occ, n, seed):
    rng = np.random.default_rng(seed)
    js, is_ = np.nonzero(occ == 0)
    q = rng.integers(0, len(is_), n)
    # off-centre positions inside the free cell, arbitrary headings
    return np.stack([is_[q] * 0.1 + rng.uniform(0.01, 0.09, n), js[q] * 0.1 + rng.uniform(0.01, 0.09, n),
                     rng.uniform(-math.pi, math.pi, n)], axis=1)


@pytest.mark.parametrize("beams,fov", [(24, 2 * math.pi), (8, 2 * math.pi), (31, 1.5), (1, 0.0), (360, 2 * math.pi)])
def test_simulate_scans_noise_free_bit_exact(ctx, ref, beams, fov):
    import oracle
    occ = make_floorplan(200, 150, seed=71)
    rm = oracle.RefMap(ref, occ=occ)
    m = g.OccupancyMap(200, 150, 0.1, occ, ctx=ctx)
    poses = _free_poses(occ, 300, beams)
    angles, ranges = g.simulate_scans(m, poses, beams, fov, 8.0)
    for q, p in enumerate(poses):
        a, r = _ref_scan(ref, rm, p, beams, fov, 8.0, 0.0, 0)
        assert np.array_equal(angles.view(np.uint64), a.view(np.uint64))
        assert np.array_equal(ranges[q].view(np.uint64), r.view(np.uint64)), f"pose {q}"


def test_simulate_scan_with_noise_matches_reference_rng(ctx, ref):
    import oracle
    occ = random_map(80, 60, 0.15, 9)
    rm = oracle.RefMap(ref, occ=occ)
    m = g.OccupancyMap(80, 60, 0.1, occ, ctx=ctx)
    for q, p in enumerate(_free_poses(occ, 40, 5)):
        seed = 1000 + q
        s = g.simulate_scan(m, g.Pose2(*p), 24, 2 * math.pi, 3.0, 0.05, rng=Rng(seed))
        a, r = _ref_scan(ref, rm, p, 24, 2 * math.pi, 3.0, 0.05, seed)
        assert np.array_equal(s.ranges.view(np.uint64), r.view(np.uint64)), f"pose {q}"


def test_raycast_corner_ties_and_axes(ctx, ref):
    """45-degree and axis-aligned beams from cell centres: the reference's
    tie tolerance advances both axes at a corner."""
    import oracle
    occ = random_map(64, 64, 0.2, 4)
    rm = oracle.RefMap(ref, occ=occ)
    m = g.OccupancyMap(64, 64, 0.1, occ, ctx=ctx)
    js, is_ = np.nonzero(occ == 0)
    rays, want = [], []
    for q in range(0, len(is_), 7):
        x, y = is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05
        for k in range(8):
            rays.append((x, y, k * math.pi / 4))
        a, r = _ref_scan(ref, rm, (x, y, 0.0), 8, 2 * math.pi, 5.0, 0.0, 0)
        # the reference's beam angles are -pi + b*pi/4; reorder to k*pi/4
        want.extend([r[(k + 4) % 8] for k in range(8)])
    got = g.raycast(m, [(x, y, -math.pi + ((k + 4) % 8) * (math.pi / 4)) for (x, y, _), k in
                        zip(rays, [i % 8 for i in range(len(rays))])], 5.0)
    assert np.array_equal(got.view(np.uint64), np.array(want).view(np.uint64))


def test_errors_like_the_reference(ctx):
    occ = make_floorplan(64, 48, seed=3)
    m = g.OccupancyMap(64, 48, 0.1, occ, ctx=ctx)
    js, is_ = np.nonzero(occ != 0)
    wall = (is_[0] * 0.1 + 0.05, js[0] * 0.1 + 0.05, 0.0)
    with pytest.raises(g.MapParseError):
        g.simulate_scans(m, [wall], 8, 2 * math.pi, 8.0)
    with pytest.raises(g.MapParseError):
        g.raycast(m, [wall], 8.0)
    free = _free_poses(occ, 1, 1)
    with pytest.raises(ValueError):
        g.simulate_scans(m, free, 0, 2 * math.pi, 8.0)
    with pytest.raises(ValueError):
        g.raycast(m, free, 0.0)
    with pytest.raises(ValueError):
        g.simulate_scans(m, free, 8, 2 * math.pi, 8.0, range_noise_sigma=0.1)  # no rng for the draws
