"""The single-process multi-device engine (gl_engine_*, engine.cpp): a
theta-slab sharded belief driven from ONE process over a device list — the
C++ callers' multi-GPU path (SURVEY.md §8(b) device list, §8(e)). This box
has one GPU, so the device list repeats device 0 (shards then share it; the
halo reads and the P2P max gather are the same code, over local instead of
NVLink memory); the NCCL reduction mode is exercised with a one-device
communicator. Every step, observation, argmax and hash must be bitwise the
unsharded tensor's (sharding changes no per-element operation)."""
import math

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from paper_1910_00572_b200._lib import GL_ENGINE_NCCL, GL_ENGINE_P2P
from tests.helpers import Rng, assert_bitwise, make_floorplan, random_motion

pytestmark = pytest.mark.gpu


def _scan(occ, q_frac=0.5, th=0.4):
    from paper_1910_00572_b200.floorplan import simple_scan
    js, is_ = np.nonzero(occ == 0)
    q = int(len(is_) * q_frac)
    a, r = simple_scan(occ, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, th)
    return g.LidarScan(a, r, 8.0)


@pytest.mark.parametrize("devices,channels,mode", [([0, 0], 72, GL_ENGINE_P2P), ([0, 0, 0], 72, GL_ENGINE_P2P),
                                                   ([0, 0, 0, 0], 360, GL_ENGINE_P2P), ([0], 72, GL_ENGINE_NCCL),
                                                   ([0, 0, 0, 0, 0, 0, 0, 0], 72, GL_ENGINE_P2P)])
def test_engine_bitwise_equals_unsharded(ctx, devices, channels, mode):
    occ = make_floorplan(128, 96, seed=61)
    m = g.OccupancyMap(128, 96, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    dth = 2 * math.pi / channels
    ks = [g.build_kernels(g.MotionNoise(), channels, 0.1, dth),
          g.build_kernels(g.MotionNoise(1e-4, 1e-4, 0.012), channels, 0.1, dth)]
    acts = [g.make_activation(m, k, channels, ctx) for k in ks]
    t = g.init_uniform(m, channels, ctx)
    e = g.Engine(devices, m, channels, mode)
    e.set_kernels(0, ks[0])
    e.set_kernels(1, ks[1])
    e.init_uniform()
    info = e.info()
    assert info["shards"] == len(devices)
    assert info["mode"] == ("nccl" if mode == GL_ENGINE_NCCL else "p2p")
    rng = Rng(len(devices) * 7 + channels)
    for s in range(10):
        u = g.OdometryDelta(*random_motion(rng)) if s % 3 else g.OdometryDelta(0.0, 0.0, rng.uniform(-0.1, 0.1))
        slot = 0 if s % 3 else 1
        g.step(t, u, m, ks[slot], acts[slot], ctx)
        e.step(u, slot)
        assert e.hash() == t.hash(), f"step {s}"
        if s == 5:
            scan = _scan(occ)
            smp_t = g.dither_samples(t, 512)
            g.observation_update(t, smp_t, scan, m, f, g.LikelihoodParams())
            smp_e = e.observe(scan)
            assert np.array_equal(smp_e.cells, smp_t.cells) and smp_e.source_mass == smp_t.source_mass
            assert e.hash() == t.hash(), "after the observation"
    vals, th = e.values()
    assert_bitwise(vals, t.values(), "engine download")
    assert th == t.theta_t()
    assert_bitwise(e.belief_map(), g.belief_map(t), "belief map")
    ee, et = e.argmax(), g.argmax_state(t)
    assert (ee.i, ee.j, ee.k) == (et.i, et.j, et.k)
    assert (ee.pose.x, ee.pose.y, ee.pose.theta) == (et.pose.x, et.pose.y, et.pose.theta)
    assert ee.confidence == et.confidence  # the sequential total chained through the shards


def test_engine_upload_rescale_and_errors(ctx):
    """Upload of a tiny-valued belief takes the step's max < 1e-6 rescale
    branch on every shard identically; bad arguments are rejected."""
    occ = make_floorplan(96, 64, seed=62)
    m = g.OccupancyMap(96, 64, 0.1, occ, ctx=ctx)
    C = 36
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    B0 = np.random.default_rng(3).random((C, 64, 96)) * 1e-9
    B0[:, occ != 0] = 0.0
    t = g.BeliefTensor(96, 64, C, 0.1, ctx=ctx)
    t.set_values(B0)
    e = g.Engine([0, 0, 0], m, C, GL_ENGINE_P2P)
    with pytest.raises(ValueError):
        e.step(g.OdometryDelta(0.1, 0.0, 0.0))  # no kernels / tensor yet
    e.set_kernels(0, ks)
    e.init_uniform()
    e.set_values(B0, 0.0)
    for u in [(0.05, 0.0, 0.1), (0.1, 0.02, 0.0)]:
        g.step(t, g.OdometryDelta(*u), m, ks, act, ctx)
        e.step(g.OdometryDelta(*u), 0)
        assert e.hash() == t.hash()
    assert e.values()[0].max() == t.values().max()
    with pytest.raises(ValueError):
        e.step(g.OdometryDelta(0.1, 0.0, 0.0), slot=1)  # slot 1 not set
    with pytest.raises(ValueError):
        g.Engine([0, 0], m, C, GL_ENGINE_NCCL)  # NCCL needs distinct devices
