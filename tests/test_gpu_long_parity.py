"""North-star parity at the benchmark sizes, in lockstep with the UNMODIFIED
reference compiled from its own sources (oracle/_ref, all host cores):

* configs[1] blind, 1024x1024x72 floor plan, a recorded Localizer trace
  (reference simulator + trigger, both kernel slots), 1000 steps by default:
  device hash == reference hash after EVERY step (bit-exact belief, hence the
  identical argmax), argmax compared every 10 steps;
* configs[2] LIDAR, CLOSED loop: every 16 steps the GPU runs the whole
  observation on its OWN belief (belief_map -> Floyd-Steinberg(512) ->
  likelihood update) and the reference on its own; the sample lists and
  source masses must be identical, the belief bit-identical after every
  step and observation (host-glibc likelihood exp, the default), relative
  L1 <= 1e-5 and the identical argmax after every observation;
* the same observation with the device exp (gl_context_set_host_exp(0)),
  open loop on the reference's samples: <= 1e-5 relative L1, same argmax;
* configs[3]'s angular width at 1024^2: 1024x1024x360 (H = 3: 4-row tiles,
  the high-word-max path that is the default at >= 2^27 states), both slots,
  device hash == reference hash every step.

GRIDLOC_LONG_PARITY overrides the step count (default 1000). Each test
writes a JSON summary to gpurun_out/ (copied to profiles/ by hand)."""
import ctypes as C
import json
import math
import os
import time

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from tests.helpers import make_floorplan, rel_l1

pytestmark = pytest.mark.gpu

N_STEPS = int(os.environ.get("GRIDLOC_LONG_PARITY", "1000"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(ref, ctx, C_, W=1024, H=1024):
    import oracle
    occ = make_floorplan(W, H, seed=0)
    rm = oracle.RefMap(ref, occ=occ)
    eng = oracle.RefEngine(ref, rm, C_, threads=0)
    m = g.OccupancyMap(W, H, 0.1, occ, ctx=ctx)
    dth = 2 * math.pi / C_
    ks = [g.build_kernels(g.MotionNoise(), C_, 0.1, dth), g.build_kernels(g.MotionNoise(1e-4, 1e-4, 0.012), C_,
                                                                          0.1, dth)]
    acts = [g.make_activation(m, k, C_, ctx) for k in ks]
    t = g.init_uniform(m, C_, ctx)
    js, is_ = np.nonzero(occ == 0)
    q = len(is_) // 3
    start = (is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.5)
    return occ, rm, eng, m, ks, acts, t, start


def _hash(ref, eng):
    ref.lib.ref_tensor_hash.restype = C.c_uint64
    ref.lib.ref_tensor_hash.argtypes = [C.c_void_p]
    return ref.lib.ref_tensor_hash(eng.t)


def _write(name, summary):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", name), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary))


def _scan(ref, rm, occ, s):
    """A noise-free 24-beam scan (reference simulator, occupancy_map.cpp:
    273-332 raycast) from a free cell chosen by the step index."""
    import oracle
    a, r = np.zeros(24), np.zeros(24)
    js, is_ = np.nonzero(occ == 0)
    q = (s * 7919) % len(is_)
    pose = (is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.1 * s)
    ref.check(ref.lib.ref_simulate_scan(rm.h, pose[0], pose[1], pose[2], 24, 2 * math.pi, 8.0, 0.0, s,
                                        oracle._d(a), oracle._d(r)), "scan")
    return a, r


def test_blind_trace_1024x72_bit_exact(ctx, ref):
    import oracle
    occ, rm, eng, m, ks, acts, t, start = _setup(ref, ctx, 72)
    ev, _ = oracle.ref_gen_trace(ref, rm, 72, start, seed=11, max_steps=N_STEPS)
    steps = ev[ev[:, 0] == 0]
    assert len(steps) == N_STEPS
    mismatch, argmax_checked, rot = 0, 0, 0
    t0 = time.time()
    for s, e in enumerate(steps):
        slot = int(e[4])
        rot += slot
        assert eng.step(e[1], e[2], e[3], slot=slot) == 0
        g.step(t, g.OdometryDelta(e[1], e[2], e[3]), m, ks[slot], acts[slot], ctx)
        if t.hash() != _hash(ref, eng):
            mismatch += 1
        if s % 10 == 9:
            ge = g.argmax_state(t)
            (i, j, k), pose, _ = eng.argmax()
            assert (ge.i, ge.j, ge.k) == (i, j, k) and (ge.pose.x, ge.pose.y, ge.pose.theta) == pose
            argmax_checked += 1
    th = eng.get()[1]
    assert t.theta_t() == th
    summary = {"config": "1024x1024x72 floor plan, recorded Localizer trace", "steps": len(steps),
               "rotation_only_steps": rot, "hash_mismatches": mismatch, "argmax_checked": argmax_checked,
               "wall_s": time.time() - t0, "result": "bit-exact" if mismatch == 0 else "MISMATCH"}
    _write(f"parity_blind_1024x72_{len(steps)}.json", summary)
    assert mismatch == 0


def test_lidar_trace_1024x72_closed_loop(ctx, ref):
    """Config 3, closed loop: each side dithers its OWN belief."""
    import oracle
    occ, rm, eng, m, ks, acts, t, start = _setup(ref, ctx, 72)
    f = g.DistanceField(m, ctx)
    ev, _ = oracle.ref_gen_trace(ref, rm, 72, start, seed=12, max_steps=N_STEPS)
    steps = ev[ev[:, 0] == 0]
    assert len(steps) == N_STEPS
    worst, n_obs, sample_mismatch, hash_mismatch, n_samples = 0.0, 0, 0, 0, []
    t0 = time.time()
    for s, e in enumerate(steps):
        slot = int(e[4])
        assert eng.step(e[1], e[2], e[3], slot=slot) == 0
        g.step(t, g.OdometryDelta(e[1], e[2], e[3]), m, ks[slot], acts[slot], ctx)
        if s % 16 == 15:
            a, r = _scan(ref, rm, occ, s)
            cells_r, mass_r = oracle.ref_dither(ref, eng.belief_map(), 512)
            smp = g.dither_samples(t, 512)  # the GPU's own belief
            if not (np.array_equal(smp.cells, cells_r) and smp.source_mass == mass_r):
                sample_mismatch += 1
            n_samples.append(len(cells_r))
            assert eng.observation_update(cells_r, a, r, 8.0) == 0
            g.observation_update(t, smp, g.LidarScan(a, r, 8.0), m, f, g.LikelihoodParams())
            Bg, Br = t.values(), eng.get()[0]
            worst = max(worst, rel_l1(Bg, Br))
            ge = g.argmax_state(t)
            (i, j, k), _, _ = eng.argmax()
            assert (ge.i, ge.j, ge.k) == (i, j, k), f"argmax differs after observation {n_obs}"
            n_obs += 1
        if t.hash() != _hash(ref, eng):
            hash_mismatch += 1
    summary = {"config": "1024x1024x72 + LIDAR every 16 steps (budget 512), closed loop (each side dithers its own "
                         "belief)", "steps": len(steps), "observations": n_obs,
               "samples_per_observation": [min(n_samples), max(n_samples)] if n_samples else None,
               "sample_set_mismatches": sample_mismatch, "belief_hash_mismatches": hash_mismatch,
               "worst_rel_l1": worst, "wall_s": time.time() - t0,
               "result": "bit-exact" if (sample_mismatch, hash_mismatch) == (0, 0) else "MISMATCH"}
    _write(f"parity_lidar_closed_1024x72_{len(steps)}.json", summary)
    assert sample_mismatch == 0
    assert hash_mismatch == 0
    assert worst <= 1e-5


def test_lidar_device_exp_open_loop(ctx, ref):
    """The device-exp likelihood mode (<= 1 ulp per likelihood): fed the
    reference's samples, within the north star's 1e-5 relative L1 with the
    identical argmax after every observation."""
    import oracle
    n = min(N_STEPS, 320)
    occ, rm, eng, m, ks, acts, t, start = _setup(ref, ctx, 72)
    f = g.DistanceField(m, ctx)
    ev, _ = oracle.ref_gen_trace(ref, rm, 72, start, seed=14, max_steps=n)
    steps = ev[ev[:, 0] == 0]
    ctx.set_host_exp(False)
    worst, n_obs = 0.0, 0
    try:
        for s, e in enumerate(steps):
            slot = int(e[4])
            assert eng.step(e[1], e[2], e[3], slot=slot) == 0
            g.step(t, g.OdometryDelta(e[1], e[2], e[3]), m, ks[slot], acts[slot], ctx)
            if s % 16 == 15:
                a, r = _scan(ref, rm, occ, s)
                cells_r, _ = oracle.ref_dither(ref, eng.belief_map(), 512)
                assert eng.observation_update(cells_r, a, r, 8.0) == 0
                g.observation_update(t, g.SampleSet(cells_r), g.LidarScan(a, r, 8.0), m, f, g.LikelihoodParams())
                worst = max(worst, rel_l1(t.values(), eng.get()[0]))
                ge = g.argmax_state(t)
                (i, j, k), _, _ = eng.argmax()
                assert (ge.i, ge.j, ge.k) == (i, j, k)
                n_obs += 1
    finally:
        ctx.set_host_exp(True)
    _write(f"parity_lidar_devexp_1024x72_{len(steps)}.json",
           {"config": "1024x1024x72 + LIDAR every 16 steps, device exp, open loop", "steps": len(steps),
            "observations": n_obs, "worst_rel_l1": worst})
    assert worst <= 1e-5


def test_trace_1024x360_lockstep_h3(ctx, ref):
    """configs[3]'s angular stencil (Theta = 360: 7 angular taps, H = 3) at
    1024^2 (377 M states): 4-row tiles and the high-word max with the exact
    epilogue, which the product enables by default at >= 2^27 states. Four
    cmd_bench translation steps (main kernels) then a recorded trace (mostly
    the rotation-only slot); the device hash equals the reference's after
    every step."""
    import oracle
    n = int(os.environ.get("GRIDLOC_PARITY_360", "24"))
    occ, rm, eng, m, ks, acts, t, start = _setup(ref, ctx, 360)
    ev, _ = oracle.ref_gen_trace(ref, rm, 360, start, seed=21, max_steps=n - 4)
    steps = [(0, 0.1, 0.0, 0.0, 0)] * 4 + [tuple(e[:5]) for e in ev[ev[:, 0] == 0]]
    slots = [int(e[4]) for e in steps]
    assert 0 in slots and 1 in slots
    mismatch = 0
    launches = []
    t0 = time.time()
    for e in steps:
        slot = int(e[4])
        assert eng.step(e[1], e[2], e[3], slot=slot) == 0
        n0 = ctx.launch_count()
        g.step(t, g.OdometryDelta(e[1], e[2], e[3]), m, ks[slot], acts[slot], ctx)
        launches.append(ctx.launch_count() - n0)
        if t.hash() != _hash(ref, eng):
            mismatch += 1
    ge = g.argmax_state(t)
    (i, j, k), pose, _ = eng.argmax()
    assert (ge.i, ge.j, ge.k) == (i, j, k)
    assert t.theta_t() == eng.get()[1]
    # fused step + the high-word-max epilogue: two launches per step
    himax = all(x == 2 for x in launches)
    _write(f"parity_1024x360_{len(steps)}.json",
           {"config": "1024x1024x360 floor plan (H = 3), 4 translation steps + recorded trace", "steps": len(steps),
            "rotation_only_steps": int(sum(slots)), "hash_mismatches": mismatch, "himax_path": himax,
            "wall_s": time.time() - t0, "result": "bit-exact" if mismatch == 0 else "MISMATCH"})
    assert himax
    assert mismatch == 0
