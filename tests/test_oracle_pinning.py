"""Pins the CPU oracle (oracle/gl_oracle.c) before it is trusted as the GPU
checker: bit-exact against the UNMODIFIED reference compiled from
/root/reference (oracle/_ref), plus the reference's own known-answer tests
(proj/tests/test_belief_engine.cpp, test_observation.cpp) run on the oracle.
CPU only."""
import math

import numpy as np
import pytest

import oracle
from tests.helpers import (Rng, assert_bitwise, make_empty_room, make_floorplan, random_map, random_motion,
                           twin_room_map)

NOISES = [
    ((0.03, 0.03, 0.012), 72),   # Localizer defaults at config-2 channels
    ((0.03, 0.03, 0.012), 36),   # config 1 (angular degenerate)
    ((0.03, 0.03, 0.012), 360),  # config 4 (7 angular taps)
    ((0.06, 0.05, 0.07), 8),     # test_belief_engine.cpp:425-449 inputs (anisotropic r=2)
    ((0.05, 0.05, 2.0), 8),      # folded angular (test :195-201)
    ((0.3, 0.2, 0.1), 12),       # generic dense interior order (r = 9)
    ((0.06, 0.06, 0.08), 8),     # isotropic r = 2
]


@pytest.mark.parametrize("noise,C", NOISES)
def test_step_bitexact_vs_reference(port, ref, noise, C):
    occ = make_floorplan(96, 72, seed=1)
    rm = oracle.RefMap(ref, occ=occ)
    eng = oracle.RefEngine(ref, rm, C, noise=noise, threads=3)
    cells = rm.cells
    rng = Rng(5)
    B, th = eng.get()
    for s in range(5):
        u = random_motion(rng)
        slot = s % 2
        rc = eng.step(*u, slot=slot)
        ks = port.build_kernels(*(noise if slot == 0 else (1e-4, 1e-4, noise[2])), C, 0.1)
        _, inv = port.make_activation(cells, ks, C)
        rcp, th = port.step(B, th, *u, cells, 0.1, ks, inv)
        Br, thr = eng.get()
        assert rc == rcp and th == thr
        assert_bitwise(B, Br, f"step {s}")


@pytest.mark.parametrize("noise,C", NOISES)
def test_kernels_and_activation_bitexact(port, ref, noise, C):
    occ = random_map(40, 30, 0.15, 3)
    rm = oracle.RefMap(ref, occ=occ)
    eng = oracle.RefEngine(ref, rm, C, noise=noise, threads=2)
    for slot, nz in enumerate([noise, (1e-4, 1e-4, noise[2])]):
        kr = eng.kernels(slot)
        kp = port.build_kernels(*nz, C, 0.1)
        assert (kr.radius, kr.separable) == (kp.radius, kp.separable)
        assert_bitwise(kr.sep, kp.sep, "sep")
        assert_bitwise(kr.spatial, kp.spatial, "spatial")
        assert list(kr.ang_off) == list(kp.ang_off)
        assert_bitwise(kr.ang_w, kp.ang_w, "angular")
        vr, ir = eng.activation(slot)
        vp, ip = port.make_activation(rm.cells, kp, C)
        assert_bitwise(vr, vp, "activation")
        assert_bitwise(ir, ip, "inverse")


def test_rescale_and_extinguish_branches_vs_reference(port, ref):
    occ = make_floorplan(64, 48, seed=2)
    rm = oracle.RefMap(ref, occ=occ)
    B0 = np.random.default_rng(1).random((16, 48, 64)) * 1e-9
    B0[:, occ != 0] = 0
    eng = oracle.RefEngine(ref, rm, 16, tensor=B0, threads=2)
    ks = port.build_kernels(0.03, 0.03, 0.012, 16, 0.1)
    _, inv = port.make_activation(rm.cells, ks, 16)
    B = B0.copy()
    rc = eng.step(0.05, 0.0, 0.1)
    rcp, th = port.step(B, 0.0, 0.05, 0.0, 0.1, rm.cells, 0.1, ks, inv)
    assert rc == rcp == 0
    assert_bitwise(B, eng.get()[0], "rescaled")
    assert B.max() == 1.0
    one = np.ones((8, 8), np.uint8)
    one[3, 3] = 0
    rm1 = oracle.RefMap(ref, occ=one)
    e1 = oracle.RefEngine(ref, rm1, 4, noise=(0.001, 0.001, 0.0001), threads=1)
    assert e1.step(0.4, 0.0, 0.0) == oracle.EXTINGUISHED
    k1 = port.build_kernels(0.001, 0.001, 0.0001, 4, 0.1)
    _, i1 = port.make_activation(rm1.cells, k1, 4)
    B1 = port.init_uniform(rm1.cells, 4)
    rc1, _ = port.step(B1, 0.0, 0.4, 0.0, 0.0, rm1.cells, 0.1, k1, i1)
    assert rc1 == oracle.EXTINGUISHED
    assert_bitwise(B1, e1.get()[0], "extinguished tensor")


def test_apply_motion_belief_map_argmax_vs_reference(port, ref):
    occ = make_floorplan(80, 60, seed=4)
    rm = oracle.RefMap(ref, occ=occ)
    B0 = np.random.default_rng(2).random((8, 60, 80))
    eng = oracle.RefEngine(ref, rm, 8, tensor=B0, threads=2)
    B = B0.copy()
    th = port.apply_motion(B, 0.0, 0.37, 0.21, 0.05, 0.1)
    eng.apply_motion(0.37, 0.21, 0.05)
    Br, thr = eng.get()
    assert th == thr
    assert_bitwise(B, Br, "apply_motion")
    assert_bitwise(port.belief_map(B), eng.belief_map(), "belief_map")
    (ijk, pose, conf) = port.argmax(B, 0.1, 0.0, 0.0, th)
    (ijk_r, pose_r, conf_r) = eng.argmax()
    assert ijk == ijk_r and pose == pose_r and conf == conf_r


def test_dither_bitexact_vs_reference(port, ref):
    rng = np.random.default_rng(3)
    for trial in range(20):
        w, h = int(rng.integers(8, 120)), int(rng.integers(8, 90))
        bm = rng.random((h, w)) * (rng.random((h, w)) < 0.7)
        budget = int(rng.integers(1, 600))
        cp, mp = port.dither(bm, budget)
        cr, mr = oracle.ref_dither(ref, bm, budget)
        assert mp == mr
        assert np.array_equal(cp, cr), trial


def test_observation_vs_reference(port, ref):
    occ = make_floorplan(120, 90, seed=6)
    rm = oracle.RefMap(ref, occ=occ)
    field = rm.field_values()
    assert_bitwise(port.distance_field(rm.cells, 0.1), field, "distance_field")
    ks = port.build_kernels(0.03, 0.03, 0.012, 16, 0.1)
    eng = oracle.RefEngine(ref, rm, 16, threads=2)
    B, th = eng.get()
    for _ in range(3):
        eng.step(0.1, 0.0, 0.05)
    B, th = eng.get()
    js, is_ = np.nonzero(occ == 0)
    pose = (is_[100] * 0.1 + 0.05, js[100] * 0.1 + 0.05, 0.4)
    ang, rng_ = np.zeros(24), np.zeros(24)
    import ctypes as C
    ref.check(ref.lib.ref_simulate_scan(rm.h, pose[0], pose[1], pose[2], 24, 2 * math.pi, 8.0, 0.0, 1,
                                        oracle._d(ang), oracle._d(rng_)), "scan")
    for stride in (1, 4):
        for q in range(0, len(is_), 997):
            p = (is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.3 * q)
            out = C.c_double()
            ref.check(ref.lib.ref_scan_likelihood(rm.h, rm.field, p[0], p[1], p[2], oracle._d(ang),
                                                  oracle._d(rng_), 24, 8.0, 0.2, 0.05, stride, C.byref(out)), "l")
            assert port.scan_likelihood(rm.cells, field, 0.1, 0.0, 0.0, p, ang, rng_, 8.0, 0.2, 0.05, stride) \
                == out.value
    cells, _ = port.dither(port.belief_map(B), 128)
    Bp = B.copy()
    rc = port.observation_update(Bp, 0.1, 0.0, 0.0, th, cells, ang, rng_, 8.0, rm.cells, field)
    rcr = eng.observation_update(cells, ang, rng_, 8.0)
    assert rc == rcr == 0
    assert_bitwise(Bp, eng.get()[0], "observation_update")


def test_load_map_vs_reference(port, ref):
    from paper_1910_00572_b200.floorplan import write_pgm
    occ = make_floorplan(70, 50, seed=8)
    data = write_pgm(occ)
    rm = oracle.RefMap(ref, pgm=data)
    assert np.array_equal(port.load_map(data), rm.cells)
    p2 = b"P2\n# comment\n4 3\n15\n" + b" ".join(str(v).encode() for v in [15, 0, 15, 15, 7, 15, 15, 15, 15, 14, 15, 0])
    assert np.array_equal(port.load_map(p2, 128), oracle.RefMap(ref, pgm=p2, threshold=128).cells)
    with pytest.raises(oracle.OracleError):
        port.load_map(b"P6\n1 1\n255\n\x00")


# ------------------------------------------------ reference known-answer tests
def test_kat_motion_vector(port):
    """test_belief_engine.cpp:79-102."""
    assert port.motion_vector(1.0, 0.0, 0, 0.0, math.pi / 4, 1.0) == (1.0, 0.0)
    dx, dy = port.motion_vector(1.0, 0.0, 1, 0.0, math.pi / 2, 1.0)
    assert abs(dx) < 1e-15 and abs(dy - 1.0) < 1e-15
    dx, dy = port.motion_vector(2.0, 0.0, 1, 0.0, math.pi / 6, 1.0)
    assert abs(dx - math.sqrt(3.0)) < 1e-12 and abs(dy - 1.0) < 1e-12
    dx, dy = port.motion_vector(0.3, -0.1, 0, 0.0, math.pi, 0.1)
    assert abs(dx - 3.0) < 1e-12 and abs(dy + 1.0) < 1e-12


def test_kat_apply_motion(port):
    """test_belief_engine.cpp:113-138."""
    B = np.zeros((4, 16, 16))
    B[0, 7, 5] = 2.0
    port.apply_motion(B, 0.0, 3.0, 0.0, 0.0, 1.0)
    assert B[0, 7, 8] == 2.0 and B[0, 7, 5] == 0.0 and np.count_nonzero(B) == 1
    B = np.zeros((4, 16, 16))
    B[0, 7, 5] = 1.0
    port.apply_motion(B, 0.0, 0.5, 0.0, 0.0, 1.0)
    assert abs(B[0, 7, 5] - 0.5) < 1e-15 and abs(B[0, 7, 6] - 0.5) < 1e-15
    th = port.apply_motion(np.zeros((4, 8, 8)), 0.0, 0.0, 0.0, 0.2, 1.0)
    th = port.apply_motion(np.zeros((4, 8, 8)), th, 0.0, 0.0, -0.05, 1.0)
    assert abs(th - 0.15) < 1e-15


def test_kat_uniform_fixed_point_and_mass(port):
    """test_belief_engine.cpp:203-227 and :263-281."""
    for occ in (random_map(24, 20, 0.15, 5), twin_room_map()):
        ks = port.build_kernels(0.06, 0.05, 0.06, 8, 0.1)
        _, inv = port.make_activation(occ, ks, 8)
        B = port.init_uniform(occ, 8)
        before = B.copy()
        port.step(B, 0.0, 0.0, 0.0, 0.0, occ, 0.1, ks, inv)
        nz = before != 0
        assert (B[~nz] == 0).all()
        assert np.max(np.abs(B[nz] - before[nz]) / before[nz]) < 1e-9
    occ = make_empty_room(48, 48)
    ks = port.build_kernels(0.06, 0.06, 0.05, 8, 0.1)
    _, inv = port.make_activation(occ, ks, 8)
    B = np.zeros((8, 48, 48))
    r = Rng(9)
    for k in range(8):
        for j in range(15, 33):
            for i in range(15, 33):
                B[k, j, i] = r.uniform()
    m0 = B.sum()
    port.step(B, 0.0, 0.0, 0.0, 0.0, occ, 0.1, ks, inv)
    assert abs(B.sum() - m0) <= 1e-9 * m0


def test_kat_argmax_ties_and_dither(port):
    """test_belief_engine.cpp:489-498; test_observation.cpp:36-101."""
    B = np.zeros((4, 8, 8))
    B[2, 5, 5] = B[2, 3, 3] = B[1, 6, 6] = 1.0
    (i, j, k), _, _ = port.argmax(B, 0.1, 0.0, 0.0, 0.0)
    assert (k, i, j) == (1, 6, 6)
    g = np.zeros((14, 14))
    g[2:12, 2:12] = 1.0
    cells, mass = port.dither(g, 25)
    assert abs(len(cells) - 25) <= 1 and abs(mass - 100.0) < 1e-12
    imp = np.zeros((16, 16))
    imp[8, 8] = 1.0
    cells, _ = port.dither(imp, 5)
    assert len(cells) == 1
    r = Rng(99)
    for _ in range(20):
        gg = np.zeros((18, 24))
        flat = gg.reshape(-1)
        for q in range(flat.size):
            flat[q] = r.uniform() if r.uniform() < 0.7 else 0.0
        budget = 8 + int(r.uniform_int(120))
        cells, _ = port.dither(gg, budget)
        assert abs(len(cells) - budget) <= 1
        assert len({tuple(c) for c in cells}) == len(cells)
        assert all(gg[c[1], c[0]] > 0 for c in cells)
