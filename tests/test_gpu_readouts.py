"""GPU parity of the read-outs and the observation path against the CPU
oracle: make_activation, apply_motion, belief_map, argmax_state (tie rule),
the tensor hash, dither_samples (bit-exact sample list, incl. on the
reference's own belief), scan_likelihood and observation_update."""
import math

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from tests.helpers import Rng, assert_bitwise, make_empty_room, make_floorplan, random_map, rel_l1, twin_room_map

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("noise,C", [((0.03, 0.03, 0.012), 72), ((0.06, 0.05, 0.07), 8),
                                     ((0.05, 0.05, 2.0), 8), ((1e-4, 1e-4, 0.012), 36)])
def test_activation_bit_exact(ctx, port, noise, C):
    occ = make_floorplan(90, 70, seed=2)
    m = g.OccupancyMap(90, 70, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(*noise), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    pk = port.build_kernels(*noise, C, 0.1)
    vals, inv = port.make_activation(m.cells(), pk, C)
    assert_bitwise(act.values, vals, "activation values")
    assert_bitwise(act.inverse, inv, "activation inverse")


def test_apply_motion_bit_exact(ctx, port):
    occ = make_floorplan(64, 48, seed=3)
    B0 = np.random.default_rng(4).random((8, 48, 64))
    t = g.BeliefTensor(64, 48, 8, 0.1, ctx=ctx)
    t.set_values(B0)
    B = B0.copy()
    th = 0.0
    for (u, v, w) in [(0.37, 0.21, 0.05), (0.0, 0.0, 0.3), (0.1, 0.0, 0.0), (-0.25, 0.4, -0.1)]:
        g.apply_motion(t, g.OdometryDelta(u, v, w))
        th = port.apply_motion(B, th, u, v, w, 0.1)
        assert t.theta_t() == th
        assert_bitwise(t.values(), B, "apply_motion")


def test_belief_map_argmax_hash(ctx, port):
    occ = make_floorplan(80, 60, seed=5)
    B = np.random.default_rng(6).random((16, 60, 80))
    t = g.BeliefTensor(80, 60, 16, 0.1, 0.5, -1.0, ctx=ctx)
    t.set_values(B)
    t.set_theta_t(0.7)
    assert_bitwise(g.belief_map(t), port.belief_map(B), "belief_map")
    est = g.argmax_state(t)
    (i, j, k), pose, conf = port.argmax(B, 0.1, 0.5, -1.0, 0.7)
    assert (est.i, est.j, est.k) == (i, j, k)
    assert (est.pose.x, est.pose.y, est.pose.theta) == pose
    assert est.confidence == conf  # the reference's sequential total, bit-exact (k_seqsum.cu)
    assert t.hash() == g.tensor_hash_host(B)


def test_argmax_tie_rule(ctx):
    """test_belief_engine.cpp:489-498: lowest (k, j, i) wins."""
    B = np.zeros((4, 8, 8))
    B[2, 5, 5] = B[2, 3, 3] = B[1, 6, 6] = 1.0
    t = g.BeliefTensor(8, 8, 4, 0.1, ctx=ctx)
    t.set_values(B)
    e = g.argmax_state(t)
    assert (e.k, e.i, e.j) == (1, 6, 6)
    t.set_values(np.zeros((4, 8, 8)))
    with pytest.raises(g.BeliefExtinguishedError):
        g.argmax_state(t)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_argmax_fused_chunk_pass_ties(ctx, port, seed):
    """Tensors of 2+ chunks (8192 states each) take the argmax candidates in the exact
    total's chunk pass (k_seqsum.cu k_chunk_sums): equal maxima planted in
    different chunks and inside one chunk, the lowest flat index must win,
    and the confidence stays the sequential total."""
    rng = np.random.default_rng(seed)
    B = rng.random((12, 70, 90)) * 0.5
    flat = B.reshape(-1)
    spots = np.sort(rng.choice(flat.size, 6, replace=False))
    flat[spots] = 0.75
    flat[spots[-1] - 1] = 0.75  # a tie inside one chunk too
    t = g.BeliefTensor(90, 70, 12, 0.1, 0.5, -1.0, ctx=ctx)
    t.set_values(B)
    t.set_theta_t(0.3)
    est = g.argmax_state(t)
    (i, j, k), pose, conf = port.argmax(B, 0.1, 0.5, -1.0, 0.3)
    assert (est.i, est.j, est.k) == (i, j, k)
    assert est.confidence == conf


@pytest.mark.parametrize("w,h,p", [(1, 7, 0.0), (7, 1, 0.0), (2, 2, 0.0), (33, 17, 0.1), (64, 64, 0.02),
                                   (301, 123, 0.3), (512, 384, 0.05), (130, 70, 0.6)])
def test_distance_field_on_device_bit_exact(ctx, port, w, h, p):
    """distance_field (occupancy_map.cpp:231-271) runs on the device: column
    run lengths, Felzenszwalb-Huttenlocher rows, sqrt * res — bitwise the
    CPU restatement (itself pinned to the reference) on thin, tiny, sparse
    and dense maps."""
    occ = random_map(w, h, p, w * 13 + h) if min(w, h) > 2 else np.ones((h, w), np.uint8)
    m = g.OccupancyMap(w, h, 0.05, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    want = port.distance_field(m.cells(), 0.05)
    assert_bitwise(f.values(), want, f"distance field {w}x{h}")


def test_dither_bit_exact_random_maps(ctx, port):
    rng = np.random.default_rng(7)
    for trial in range(25):
        w, h = int(rng.integers(4, 150)), int(rng.integers(2, 120))
        bm = rng.random((h, w)) * (rng.random((h, w)) < 0.7)
        budget = int(rng.integers(1, 700))
        s = g.dither_samples(bm, budget, ctx)
        cells, mass = port.dither(bm, budget)
        assert s.source_mass == mass
        assert np.array_equal(s.cells, cells), trial


def test_dither_signed_zeros_and_negatives(ctx, port):
    """The device total skips zero terms (exact: a sum started at +0.0 is
    never -0.0, and x + (+-0.0) == x otherwise); planes with -0.0, negative
    and denormal entries, widths around the 256-value staging chunks."""
    rng = np.random.default_rng(11)
    for trial, (w, h) in enumerate([(255, 9), (256, 7), (257, 8), (300, 5), (1030, 3), (33, 40)]):
        bm = rng.random((h, w)) * 2.0
        z = rng.random((h, w))
        bm[z < 0.2] = 0.0
        bm[(z >= 0.2) & (z < 0.3)] = -0.0
        bm[(z >= 0.3) & (z < 0.35)] *= -1.0
        bm[(z >= 0.35) & (z < 0.37)] = 5e-324
        budget = int(rng.integers(1, 400))
        s = g.dither_samples(bm, budget, ctx)
        cells, mass = port.dither(bm, budget)
        assert np.float64(s.source_mass).tobytes() == np.float64(mass).tobytes(), trial
        assert np.array_equal(s.cells, cells), trial


def test_dither_reference_test_cases(ctx):
    """test_observation.cpp:36-101 on the GPU path."""
    gg = np.zeros((14, 14))
    gg[2:12, 2:12] = 1.0
    s = g.dither_samples(gg, 25, ctx)
    assert abs(len(s.cells) - 25) <= 1 and abs(s.source_mass - 100.0) < 1e-12
    imp = np.zeros((16, 16))
    imp[8, 8] = 1.0
    assert len(g.dither_samples(imp, 5, ctx).cells) == 1
    z = g.dither_samples(np.zeros((8, 8)), 10, ctx)
    assert len(z.cells) == 0 and z.source_mass == 0.0
    with pytest.raises(ValueError):
        g.dither_samples(np.zeros((8, 8)), 0, ctx)


def test_dither_on_reference_belief_1024(ctx, port, ref):
    """North-star: bit-exact sample set when fed the reference's belief
    (1024^2 floor plan, 72 channels, a few reference steps, budget 512)."""
    import oracle
    occ = make_floorplan(1024, 1024, seed=0)
    rm = oracle.RefMap(ref, occ=occ)
    eng = oracle.RefEngine(ref, rm, 72, threads=0, rot_slot=False)
    for (u, v, w) in [(0.1, 0.0, 0.0), (0.05, 0.02, 0.1), (0.1, -0.03, 0.0)]:
        assert eng.step(u, v, w) == 0
    bm = eng.belief_map()
    cells_r, mass_r = oracle.ref_dither(ref, bm, 512)
    s = g.dither_samples(bm, 512, ctx)
    assert s.source_mass == mass_r
    assert np.array_equal(s.cells, cells_r)
    # and from the device tensor holding the reference's belief
    B, th = eng.get()
    t = g.BeliefTensor(1024, 1024, 72, 0.1, ctx=ctx)
    t.set_values(B)
    s2 = g.dither_samples(t, 512)
    assert np.array_equal(s2.cells, cells_r) and s2.source_mass == mass_r


def _scan(ref_, rm, pose, beams=24, max_range=8.0):
    import oracle
    a = np.zeros(beams)
    r = np.zeros(beams)
    ref_.check(ref_.lib.ref_simulate_scan(rm.h, pose[0], pose[1], pose[2], beams, 2 * math.pi, max_range, 0.0, 1,
                                          oracle._d(a), oracle._d(r)), "scan")
    return a, r


def test_scan_likelihood_matches(ctx, port, ref):
    import oracle
    occ = make_floorplan(120, 90, seed=6)
    rm = oracle.RefMap(ref, occ=occ)
    m = g.OccupancyMap(120, 90, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    assert_bitwise(f.values(), rm.field_values(), "distance field")
    js, is_ = np.nonzero(occ == 0)
    a, r = _scan(ref, rm, (is_[50] * 0.1 + 0.05, js[50] * 0.1 + 0.05, 0.2))
    field = rm.field_values()
    worst = 0.0
    for q in range(0, len(is_), 211):
        pose = (is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.37 * q)
        for stride in (1, 4):
            lp = g.LikelihoodParams(0.2, 0.05, stride)
            got = g.scan_likelihood(m, f, g.Pose2(*pose), g.LidarScan(a, r, 8.0), lp)
            want = port.scan_likelihood(rm.cells, field, 0.1, 0.0, 0.0, pose, a, r, 8.0, 0.2, 0.05, stride)
            worst = max(worst, abs(got - want) / want)
    # transcendentals: host glibc for cos/sin/exp/log tables, device exp for
    # the final geometric mean (<= 2 ulp)
    assert worst <= 1e-15
    # an occupied pose scores the floor exactly
    assert g.scan_likelihood(m, f, g.Pose2(0.05, 0.05, 0.0), g.LidarScan(a, r, 8.0)) == 0.05


def test_observation_update_matches(ctx, port, ref):
    import oracle
    occ = make_floorplan(160, 120, seed=8)
    rm = oracle.RefMap(ref, occ=occ)
    m = g.OccupancyMap(160, 120, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    eng = oracle.RefEngine(ref, rm, 36, threads=0, rot_slot=False)
    for _ in range(4):
        eng.step(0.1, 0.0, 0.05)
    B, th = eng.get()
    js, is_ = np.nonzero(occ == 0)
    a, r = _scan(ref, rm, (is_[1000] * 0.1 + 0.05, js[1000] * 0.1 + 0.05, 0.4))
    cells, _ = port.dither(port.belief_map(B), 256)
    t = g.BeliefTensor(160, 120, 36, 0.1, ctx=ctx)
    t.set_values(B)
    t.set_theta_t(th)
    g.observation_update(t, g.SampleSet(cells), g.LidarScan(a, r, 8.0), m, f, g.LikelihoodParams())
    assert eng.observation_update(cells, a, r, 8.0) == 0
    Bref = eng.get()[0]
    got = t.values()
    assert rel_l1(got, Bref) <= 1e-14
    diff = np.count_nonzero(got.view(np.uint64) != Bref.view(np.uint64))
    print("observation_update: values differing in the last bits:", diff, "of", got.size)
    e = g.argmax_state(t)
    (i, j, k), _, _ = port.argmax(Bref, 0.1, 0.0, 0.0, th)
    assert (e.i, e.j, e.k) == (i, j, k)
    # empty sample set: no-op (observation.cpp:117)
    before = t.values()
    g.observation_update(t, g.SampleSet(np.zeros((0, 2), np.int32)), g.LidarScan(a, r, 8.0), m, f)
    assert_bitwise(t.values(), before, "no-op")


def test_tensors_status_batch(ctx):
    """gl_tensors_status: many tensors' latest step status in one round trip;
    an extinguished one raises like gl_tensor_status."""
    import math
    occ = make_floorplan(40, 30, seed=3)
    m = g.OccupancyMap(40, 30, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), 8, 0.1, 2 * math.pi / 8)
    act = g.make_activation(m, ks, 8, ctx)
    ts = [g.init_uniform(m, 8, ctx) for _ in range(70)]  # > 64: two gather launches
    for t in ts:
        g.step_async(t, g.OdometryDelta(0.1, 0.0, 0.0), m, ks, act, ctx)
    g.tensors_status(ts, ctx)
    ts[67].set_values(np.zeros((8, 30, 40)))
    g.step_async(ts[67], g.OdometryDelta(0.1, 0.0, 0.0), m, ks, act, ctx)
    with pytest.raises(g.BeliefExtinguishedError):
        g.tensors_status(ts, ctx)
