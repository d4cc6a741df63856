"""North-star parity at the benchmark size (BASELINE configs[1] / [2]):
1024x1024x72 floor plan, a recorded Localizer trace (reference simulator +
trigger, both kernel slots) run in lockstep on the GPU and on the compiled
reference (all host cores).

* blind trace: device hash == reference hash after EVERY step (bit-exact
  belief, hence identical argmax), argmax compared every 10 steps;
* LIDAR trace (config 3): an observation (belief_map -> Floyd-Steinberg ->
  likelihood update) after every 16 steps; relative L1 <= 1e-5 and the
  identical argmax after every observation.

Default length 200 steps (CI); GRIDLOC_LONG_PARITY=1000 runs the full
north-star length. A JSON summary is written to gpurun_out/ (copied to
profiles/ by hand)."""
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

N_STEPS = int(os.environ.get("GRIDLOC_LONG_PARITY", "200"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(ref, ctx, C_):
    import oracle
    occ = make_floorplan(1024, 1024, seed=0)
    rm = oracle.RefMap(ref, occ=occ)
    eng = oracle.RefEngine(ref, rm, C_, threads=0)
    m = g.OccupancyMap(1024, 1024, 0.1, occ, ctx=ctx)
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


def test_lidar_trace_1024x72(ctx, ref):
    """Config 3: odometry + map steps and, every 16 steps, a sampled LIDAR
    update (belief_map -> dither_samples(512) -> observation_update)."""
    import oracle
    occ, rm, eng, m, ks, acts, t, start = _setup(ref, ctx, 72)
    f = g.DistanceField(m, ctx)
    ev, scans = oracle.ref_gen_trace(ref, rm, 72, start, seed=12, max_steps=N_STEPS)
    steps = ev[ev[:, 0] == 0]
    worst, n_obs, sample_mismatch = 0.0, 0, 0
    t0 = time.time()
    for s, e in enumerate(steps):
        slot = int(e[4])
        assert eng.step(e[1], e[2], e[3], slot=slot) == 0
        g.step(t, g.OdometryDelta(e[1], e[2], e[3]), m, ks[slot], acts[slot], ctx)
        if s % 16 == 15:
            # a noise-free 24-beam scan from a free cell (reference simulator)
            a, r = np.zeros(24), np.zeros(24)
            js, is_ = np.nonzero(occ == 0)
            q = (s * 7919) % len(is_)
            pose = (is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.1 * s)
            ref.check(ref.lib.ref_simulate_scan(rm.h, pose[0], pose[1], pose[2], 24, 2 * math.pi, 8.0, 0.0, s,
                                                oracle._d(a), oracle._d(r)), "scan")
            bm = eng.belief_map()
            cells_r, mass_r = oracle.ref_dither(ref, bm, 512)
            smp = g.dither_samples(t, 512)
            if not (np.array_equal(smp.cells, cells_r) and smp.source_mass == mass_r):
                sample_mismatch += 1
            assert eng.observation_update(cells_r, a, r, 8.0) == 0
            g.observation_update(t, g.SampleSet(cells_r), g.LidarScan(a, r, 8.0), m, f, g.LikelihoodParams())
            Bg, Br = t.values(), eng.get()[0]
            worst = max(worst, rel_l1(Bg, Br))
            ge = g.argmax_state(t)
            (i, j, k), _, _ = eng.argmax()
            assert (ge.i, ge.j, ge.k) == (i, j, k), f"argmax differs after observation {n_obs}"
            n_obs += 1
    summary = {"config": "1024x1024x72 + LIDAR every 16 steps (budget 512)", "steps": len(steps),
               "observations": n_obs, "worst_rel_l1": worst, "sample_set_mismatch_vs_reference_belief":
                   sample_mismatch, "wall_s": time.time() - t0}
    _write(f"parity_lidar_1024x72_{len(steps)}.json", summary)
    assert worst <= 1e-5
