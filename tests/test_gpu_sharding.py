"""theta-slab sharding on the device: G shards of one belief held on ONE GPU
(the only GPU this build has), stepped with the sharded kernel, their step
maxima max-reduced and their halo planes exchanged by device copies along
the same HaloPlan the NCCL path uses. The concatenated interiors must be
bitwise the unsharded tensor after every step (sharding changes no
per-element operation). The multi-process NCCL/gloo plumbing is covered by
tests/test_sharding_gloo.py."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from paper_1910_00572_b200._lib import check
from paper_1910_00572_b200.sharding import halo_plan, partition
from tests.helpers import Rng, assert_bitwise, make_floorplan, random_motion

pytestmark = pytest.mark.gpu


def _shard(ctx, m, c_total, c0, c1, halo):
    h = C.c_void_p()
    check(ctx.lib.gl_shard_init_uniform(ctx.h, m.h, c_total, c0, c1, halo, C.byref(h)))
    return g.BeliefTensor(ctx=ctx, _handle=h)


def _max_bits(ctx, t):
    p = C.POINTER(C.c_uint64)()
    check(ctx.lib.gl_tensor_max_ptr(ctx.h, t.h, C.byref(p)))
    return p


@pytest.mark.parametrize("G,c_total,noise", [(2, 72, (0.03, 0.03, 0.012)), (4, 72, (0.03, 0.03, 0.012)),
                                             (3, 36, (1e-4, 1e-4, 0.012)), (8, 360, (0.03, 0.03, 0.012))])
def test_sharded_steps_bitwise_equal_unsharded(ctx, G, c_total, noise):
    import torch
    occ = make_floorplan(128, 96, seed=21)
    m = g.OccupancyMap(128, 96, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(*noise), c_total, 0.1, 2 * math.pi / c_total)
    act = g.make_activation(m, ks, c_total, ctx)
    H = len(ks.angular) // 2
    halo = max(H, 1)
    full = g.init_uniform(m, c_total, ctx)
    shards = [_shard(ctx, m, c_total, *partition(c_total, G, r), halo) for r in range(G)]
    plans = [halo_plan(c_total, G, r, halo) for r in range(G)]
    rng = Rng(G * 100 + c_total)
    motions = [random_motion(rng) for _ in range(5)] + [(0.1, 0.0, 0.0), (0.0, 0.0, 0.2)]
    for (u, v, w) in motions:
        g.step(full, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        for t in shards:
            g.step_async(t, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        ctx.synchronize()
        # all-reduce MAX of the uint64 bit patterns (emulated on one device)
        dev = [torch.as_tensor(_cai(C.cast(_max_bits(ctx, t), C.c_void_p).value), device="cuda")
               for t in shards]
        gmax = torch.stack(dev).max()
        for d in dev:
            d.copy_(gmax.reshape(1))
        torch.cuda.synchronize()
        for t in shards:
            check(ctx.lib.gl_shard_finalize(ctx.h, t.h))
        # halo exchange along the NCCL plan, as device copies
        for r, t in enumerate(shards):
            pl = plans[r]
            left, right = shards[pl.left], shards[pl.right]
            lp, rp = plans[pl.left], plans[pl.right]
            check(ctx.lib.gl_tensor_copy_planes(ctx.h, t.h, pl.recv_left[0], left.h, lp.send_right[0], halo))
            check(ctx.lib.gl_tensor_copy_planes(ctx.h, t.h, pl.recv_right[0], right.h, rp.send_left[0], halo))
        ctx.synchronize()
        for t in shards:
            g.tensor_status(t)
        got = np.concatenate([t.values() for t in shards], axis=0)
        assert_bitwise(got, full.values(), f"G={G} sharded vs unsharded")
        assert all(t.theta_t() == full.theta_t() for t in shards)


def _cai(ptr):
    class _V:
        __cuda_array_interface__ = {"shape": (1,), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                    "strides": None, "stream": None}
    return _V()


@pytest.mark.parametrize("G,c_total,noise", [(1, 72, (0.03, 0.03, 0.012)), (2, 72, (0.03, 0.03, 0.012)),
                                             (3, 36, (1e-4, 1e-4, 0.012)), (8, 360, (0.03, 0.03, 0.012))])
def test_fused_peer_halo_reads_bitwise_equal_unsharded(ctx, G, c_total, noise):
    """Peer mode: each shard's fused step TMA-reads its halo input planes
    straight from the neighbours' buffers (gl_shard_set_peers; here the
    neighbours' buffers on the same device stand in for CUDA-IPC mappings of
    other GPUs' buffers — the kernel code is the same). No exchange step
    runs and the shards' own halo planes are never written, yet every step
    must equal the unsharded belief bit for bit. G = 1 reads its own
    interior planes circularly."""
    import torch
    from paper_1910_00572_b200.sharding import peer_plan
    occ = make_floorplan(128, 96, seed=22)
    m = g.OccupancyMap(128, 96, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(*noise), c_total, 0.1, 2 * math.pi / c_total)
    act = g.make_activation(m, ks, c_total, ctx)
    halo = max(len(ks.angular) // 2, 1)
    full = g.init_uniform(m, c_total, ctx)
    shards = [_shard(ctx, m, c_total, *partition(c_total, G, r), halo) for r in range(G)]

    def base(t, b):
        p = C.POINTER(C.c_double)()
        check(ctx.lib.gl_tensor_buffer_ptr(ctx.h, t.h, b, 0, C.byref(p)))
        return C.cast(p, C.c_void_p)

    for r, t in enumerate(shards):
        pp = peer_plan(c_total, G, r, halo)
        lo, hi = shards[pp.lo_rank], shards[pp.hi_rank]
        check(ctx.lib.gl_shard_set_peers(ctx.h, t.h, base(lo, 0), base(lo, 1), pp.lo_count,
                                         base(hi, 0), base(hi, 1), pp.hi_count))
        # poison the own halo planes: peer mode must never read them
        for b in (0, 1):
            for q in list(range(halo)) + list(range(halo + t.channels(), 2 * halo + t.channels())):
                p = C.POINTER(C.c_double)()
                check(ctx.lib.gl_tensor_buffer_ptr(ctx.h, t.h, b, q, C.byref(p)))
                torch.as_tensor(_cai_f64(C.cast(p, C.c_void_p).value, 128 * 96), device="cuda").fill_(float("nan"))
    torch.cuda.synchronize()
    rng = Rng(G * 7 + c_total)
    motions = [random_motion(rng) for _ in range(5)] + [(0.1, 0.0, 0.0), (0.0, 0.0, 0.2)]
    for (u, v, w) in motions:
        g.step(full, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        for t in shards:
            g.step_async(t, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        ctx.synchronize()
        dev = [torch.as_tensor(_cai(C.cast(_max_bits(ctx, t), C.c_void_p).value), device="cuda")
               for t in shards]
        gmax = torch.stack(dev).max()
        for d in dev:
            d.copy_(gmax.reshape(1))
        torch.cuda.synchronize()
        for t in shards:
            check(ctx.lib.gl_shard_finalize(ctx.h, t.h))
        ctx.synchronize()
        for t in shards:
            g.tensor_status(t)
        got = np.concatenate([t.values() for t in shards], axis=0)
        assert_bitwise(got, full.values(), f"G={G} peer-read shards vs unsharded")


def _cai_f64(ptr, n):
    class _V:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None, "stream": None}
    return _V()
