"""The wall-crossing mask (BASELINE north star kernel (2); an EXTENSION the
reference does not have, so it is opt-in per context and every reference
parity run keeps it off): a bilinear tap whose straight segment between
source and destination cell centres crosses an occupied cell's interior is
dropped (paper_1910_00572_b200/csrc/wall.hpp). Checked bit-for-bit against
the oracle's restatement of the same rule (oracle/gl_oracle.c
glo_step_wall) on the fused kernel (the per-warp occupancy window in its
shift stage) and on the generic chain, plus the property the rule exists
for: no mass crosses a one-cell wall however far a step moves."""
import math

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from paper_1910_00572_b200._lib import GL_PATH_AUTO, GL_PATH_FUSED, GL_PATH_GENERIC
from tests.helpers import Rng, assert_bitwise, make_floorplan, random_map, random_motion, random_tensor

pytestmark = pytest.mark.gpu


def _pair(ctx, port, occ, channels, noise, motions, path, B0=None, fast=True):
    ctx.set_path(path)
    ctx.set_wall_mask(True)
    ctx.set_fast(fast)
    try:
        h, w = occ.shape
        m = g.OccupancyMap(w, h, 0.1, occ, ctx=ctx)
        ks = g.build_kernels(g.MotionNoise(*noise), channels, 0.1, 2 * math.pi / channels)
        act = g.make_activation(m, ks, channels, ctx)
        cells = m.cells()
        pks = port.build_kernels(*noise, channels, 0.1)
        _, pinv = port.make_activation(cells, pks, channels)
        if B0 is None:
            t = g.init_uniform(m, channels, ctx)
            B = port.init_uniform(cells, channels)
        else:
            t = g.BeliefTensor(w, h, channels, 0.1, ctx=ctx)
            t.set_values(B0)
            B = np.array(B0, dtype=np.float64, copy=True)
        th = 0.0
        for s, (u, v, w_) in enumerate(motions):
            rc, th = port.step(B, th, u, v, w_, cells, 0.1, pks, pinv, wall=True)
            assert rc == 0
            g.step(t, g.OdometryDelta(u, v, w_), m, ks, act, ctx)
            assert t.theta_t() == th
            assert_bitwise(t.values(), B, f"wall step {s} path {path}")
        return t, B
    finally:
        ctx.set_wall_mask(False)
        ctx.set_path(GL_PATH_AUTO)
        ctx.set_fast(True)


MOTIONS = [(0.1, 0.0, 0.0), (0.25, 0.13, 0.05), (-0.31, 0.22, -0.1), (0.0, 0.0, 0.2), (0.2, 0.2, 0.0),
           (0.35, -0.27, 0.3), (0.0, -0.2, 0.0)]


@pytest.mark.parametrize("path", [GL_PATH_FUSED, GL_PATH_GENERIC])
@pytest.mark.parametrize("channels,noise", [(72, (0.03, 0.03, 0.012)), (360, (0.03, 0.03, 0.012)),
                                            (36, (1e-4, 1e-4, 0.012)), (16, (0.06, 0.06, 0.08))])
def test_wall_mask_bit_exact_vs_oracle(ctx, port, path, channels, noise):
    occ = make_floorplan(96, 80, seed=8)
    _pair(ctx, port, occ, channels, noise, MOTIONS, path)


@pytest.mark.parametrize("fast", [True, False])
def test_wall_mask_unclean_and_random_maps(ctx, port, fast):
    """Random clutter (many thin walls), unclean uploads (negatives, -0.0)
    for the strict variant, integral shifts included."""
    occ = random_map(64, 48, 0.25, 3)
    B0 = random_tensor(occ, 72, seed=9, free_only=False)
    if not fast:
        B0 = B0 - 0.2
        B0[3, 5:9, 5:9] = -0.0
    rng = Rng(4)
    motions = [random_motion(rng, 0.4, 0.4, 0.2) for _ in range(4)] + [(0.2, 0.0, 0.0), (0.1, 0.1, 0.0)]
    _pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED, B0=B0, fast=fast)


def test_wall_mask_large_motion_takes_generic_chain(ctx, port):
    """|floor(d)| > 7 cells does not fit the fused kernel's table: AUTO runs
    the generic chain, still bit-exact."""
    occ = make_floorplan(96, 80, seed=2)
    _pair(ctx, port, occ, 36, (0.03, 0.03, 0.012), [(0.95, 0.4, 0.0), (0.1, 0.0, 0.0)], GL_PATH_AUTO)


def test_no_mass_crosses_a_one_cell_wall(ctx):
    """Two rooms split by a one-cell wall; all mass starts in the left room.
    A 2.5-cell step to the right jumps the wall without the mask (the
    reference's behaviour) and never with it."""
    W, H, C = 40, 24, 8
    occ = np.zeros((H, W), np.uint8)
    occ[0, :] = occ[-1, :] = 1
    occ[:, 0] = occ[:, -1] = 1
    occ[:, 20] = 1  # the wall
    m = g.OccupancyMap(W, H, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(1e-4, 1e-4, 0.012), C, 0.1, 2 * math.pi / C)  # no spatial diffusion
    act = g.make_activation(m, ks, C, ctx)
    B0 = np.zeros((C, H, W))
    B0[:, 1:-1, 1:20] = 1.0
    results = {}
    for wall in (False, True):
        ctx.set_wall_mask(wall)
        try:
            t = g.BeliefTensor(W, H, C, 0.1, ctx=ctx)
            t.set_values(B0)
            # channel 0 faces +x: the step moves its mass 2.5 cells right
            g.step(t, g.OdometryDelta(0.25, 0.0, 0.0), m, ks, act, ctx)
            results[wall] = t.values()[0, :, 21:].sum()
        finally:
            ctx.set_wall_mask(False)
    assert results[False] > 0.0
    assert results[True] == 0.0


def test_wall_mask_sharded_equals_unsharded(ctx):
    """theta-slab shards with the mask on (the fused kernel is the only
    sharded path) are bitwise the unsharded tensor."""
    import ctypes as C_
    import torch
    from paper_1910_00572_b200._lib import check
    from paper_1910_00572_b200.sharding import halo_plan, partition
    occ = make_floorplan(128, 96, seed=5)
    m = g.OccupancyMap(128, 96, 0.1, occ, ctx=ctx)
    c_total, G = 72, 3
    ks = g.build_kernels(g.MotionNoise(), c_total, 0.1, 2 * math.pi / c_total)
    act = g.make_activation(m, ks, c_total, ctx)
    halo = 1
    ctx.set_wall_mask(True)
    try:
        full = g.init_uniform(m, c_total, ctx)
        shards = []
        for r in range(G):
            h = C_.c_void_p()
            check(ctx.lib.gl_shard_init_uniform(ctx.h, m.h, c_total, *partition(c_total, G, r), halo, C_.byref(h)))
            shards.append(g.BeliefTensor(ctx=ctx, _handle=h))
        plans = [halo_plan(c_total, G, r, halo) for r in range(G)]
        for (u, v, w) in MOTIONS:
            g.step(full, g.OdometryDelta(u, v, w), m, ks, act, ctx)
            for t in shards:
                g.step_async(t, g.OdometryDelta(u, v, w), m, ks, act, ctx)
            ctx.synchronize()
            ptrs = []
            for t in shards:
                p = C_.POINTER(C_.c_uint64)()
                check(ctx.lib.gl_tensor_max_ptr(ctx.h, t.h, C_.byref(p)))
                ptrs.append(C_.cast(p, C_.c_void_p).value)
            # max all-reduce of the uint64 step maxima, emulated on the device
            dev = [torch.as_tensor(_CAI(p), device="cuda") for p in ptrs]
            gm = torch.stack(dev).max()
            for d in dev:
                d.copy_(gm.reshape(1))
            torch.cuda.synchronize()
            for t in shards:
                check(ctx.lib.gl_shard_finalize(ctx.h, t.h))
            for r, t in enumerate(shards):
                pl = plans[r]
                left, right = shards[pl.left], shards[pl.right]
                lp, rp = plans[pl.left], plans[pl.right]
                check(ctx.lib.gl_tensor_copy_planes(ctx.h, t.h, pl.recv_left[0], left.h, lp.send_right[0], halo))
                check(ctx.lib.gl_tensor_copy_planes(ctx.h, t.h, pl.recv_right[0], right.h, rp.send_left[0], halo))
            ctx.synchronize()
        whole = full.values()
        for r, t in enumerate(shards):
            c0, c1 = partition(c_total, G, r)
            assert_bitwise(t.values(), whole[c0:c1], f"shard {r}")
    finally:
        ctx.set_wall_mask(False)


class _CAI:
    def __init__(self, ptr):
        self.__cuda_array_interface__ = {"shape": (1,), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}
