"""configs[4] under concurrency: independent robots stepped on concurrent
contexts (one CUDA stream each), driven from concurrent host threads — the
batch engine's shape (bench.py --config c5: 64 robots on 8 streams, one
channel chunk). Per-context state (the mapped pinned status word, the misc
scratch the read-outs and observations use, the motion upload ring, the
thread-local launch parameters) must never leak between contexts: every
robot's belief must equal the reference's after every step and observation
(hash of the FP64 bits), and its Floyd-Steinberg samples must be identical.

The reference side runs afterwards, robot by robot, on the compiled
reference (oracle/_ref) with the same maps, motions and scans."""
import math
import threading

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from tests.helpers import Rng, make_floorplan, random_motion

pytestmark = pytest.mark.gpu

N_CTX, PER_CTX, W, C_, STEPS, OBS_AT = 8, 2, 512, 72, 12, 6


def _ref_hash(ref, eng):
    import ctypes as C
    ref.lib.ref_tensor_hash.restype = C.c_uint64
    ref.lib.ref_tensor_hash.argtypes = [C.c_void_p]
    return ref.lib.ref_tensor_hash(eng.t)


def test_concurrent_contexts_batch_parity(ref):
    import oracle
    ctxs = [g.Context(0) for _ in range(N_CTX)]
    for c in ctxs:
        c.set_channel_chunks(1)
    robots = []
    for r in range(N_CTX * PER_CTX):
        ctx = ctxs[r // PER_CTX]
        occ = make_floorplan(W, W, seed=100 + r)
        m = g.OccupancyMap(W, W, 0.1, occ, ctx=ctx)
        dth = 2 * math.pi / C_
        ks = [g.build_kernels(g.MotionNoise(), C_, 0.1, dth),
              g.build_kernels(g.MotionNoise(1e-4, 1e-4, 0.012), C_, 0.1, dth)]
        acts = [g.make_activation(m, k, C_, ctx) for k in ks]
        rng = Rng(500 + r)
        motions = [random_motion(rng) if s % 3 else (0.0, 0.0, rng.uniform(-0.1, 0.1)) for s in range(STEPS)]
        slots = [0 if s % 3 else 1 for s in range(STEPS)]
        js, is_ = np.nonzero(occ == 0)
        rm = oracle.RefMap(ref, occ=occ)
        a, rr = np.zeros(24), np.zeros(24)
        q = (r * 7919) % len(is_)
        ref.check(ref.lib.ref_simulate_scan(rm.h, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.3 * r, 24,
                                            2 * math.pi, 8.0, 0.0, r, oracle._d(a), oracle._d(rr)), "scan")
        robots.append(dict(ctx=ctx, occ=occ, m=m, ks=ks, acts=acts, t=g.init_uniform(m, C_, ctx),
                           f=g.DistanceField(m, ctx), motions=motions, slots=slots, scan=(a, rr), rm=rm,
                           hashes=[], samples=None, error=None))

    def drive(ci):
        mine = robots[ci * PER_CTX:(ci + 1) * PER_CTX]
        try:
            for s in range(STEPS):
                for rb in mine:  # both robots' steps in flight on this context's stream
                    u = g.OdometryDelta(*rb["motions"][s])
                    sl = rb["slots"][s]
                    g.step_async(rb["t"], u, rb["m"], rb["ks"][sl], rb["acts"][sl], rb["ctx"])
                for rb in mine:
                    g.tensor_status(rb["t"])
                    rb["hashes"].append(rb["t"].hash())
                if s == OBS_AT:
                    for rb in mine:
                        smp = g.dither_samples(rb["t"], 512, rb["ctx"])
                        g.observation_update(rb["t"], smp, g.LidarScan(*rb["scan"], 8.0), rb["m"], rb["f"],
                                             g.LikelihoodParams())
                        rb["samples"] = (smp.cells.copy(), smp.source_mass)
                        rb["hashes"].append(rb["t"].hash())
        except Exception as e:  # surfaced below
            for rb in mine:
                rb["error"] = repr(e)

    threads = [threading.Thread(target=drive, args=(ci,)) for ci in range(N_CTX)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for r, rb in enumerate(robots):
        assert rb["error"] is None, f"robot {r}: {rb['error']}"

    for r, rb in enumerate(robots):
        eng = oracle.RefEngine(ref, rb["rm"], C_, threads=0)
        want = []
        for s in range(STEPS):
            assert eng.step(*rb["motions"][s], slot=rb["slots"][s]) == 0
            want.append(_ref_hash(ref, eng))
            if s == OBS_AT:
                cells, mass = oracle.ref_dither(ref, eng.belief_map(), 512)
                got_cells, got_mass = rb["samples"]
                assert np.array_equal(got_cells, cells) and got_mass == mass, f"robot {r}: samples differ"
                assert eng.observation_update(cells, *rb["scan"], 8.0) == 0
                want.append(_ref_hash(ref, eng))
        assert rb["hashes"] == want, f"robot {r}: belief differs at " \
                                     f"{[i for i, (x, y) in enumerate(zip(rb['hashes'], want)) if x != y][:5]}"
        del eng
