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


@pytest.mark.parametrize("G,c_total,noise,W", [(1, 72, (0.03, 0.03, 0.012), 128), (2, 72, (0.03, 0.03, 0.012), 128),
                                               (3, 36, (1e-4, 1e-4, 0.012), 128), (8, 360, (0.03, 0.03, 0.012), 128),
                                               (2, 72, (0.03, 0.03, 0.012), 127),   # odd W: cp.async loads
                                               (3, 360, (0.03, 0.03, 0.012), 95)])
def test_fused_peer_halo_reads_bitwise_equal_unsharded(ctx, G, c_total, noise, W):
    """Peer mode: each shard's fused step TMA-reads its halo input planes
    straight from the neighbours' buffers (gl_shard_set_peers; here the
    neighbours' buffers on the same device stand in for CUDA-IPC mappings of
    other GPUs' buffers — the kernel code is the same). No exchange step
    runs and the shards' own halo planes are never written, yet every step
    must equal the unsharded belief bit for bit. G = 1 reads its own
    interior planes circularly."""
    import torch
    from paper_1910_00572_b200.sharding import peer_plan
    occ = make_floorplan(W, 96, seed=22)
    m = g.OccupancyMap(W, 96, 0.1, occ, ctx=ctx)
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
                torch.as_tensor(_cai_f64(C.cast(p, C.c_void_p).value, W * 96), device="cuda").fill_(float("nan"))
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


def _emulate_max_allreduce(ctx, shards):
    import torch
    dev = [torch.as_tensor(_cai(C.cast(_max_bits(ctx, t), C.c_void_p).value), device="cuda") for t in shards]
    gmax = torch.stack(dev).max()
    for d in dev:
        d.copy_(gmax.reshape(1))
    torch.cuda.synchronize()


@pytest.mark.parametrize("G,c_total", [(2, 72), (3, 36), (4, 72)])
def test_sharded_observation_bitwise_equal_unsharded(ctx, G, c_total):
    """SURVEY §8(e) LIDAR path on G shards of one belief (one device standing
    in for G ranks): local belief maps max-reduced -> dither on the reduced
    device plane -> the same samples everywhere -> every shard's likelihoods
    over all channels, own channels multiplied, max all-reduced, 1/max
    finalised. Samples, source mass and the tensor (incl. the pending
    rescale, seen through a following step) bitwise the unsharded path."""
    import torch
    from paper_1910_00572_b200.floorplan import simple_scan
    occ = make_floorplan(128, 96, seed=31)
    m = g.OccupancyMap(128, 96, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    ks = g.build_kernels(g.MotionNoise(), c_total, 0.1, 2 * math.pi / c_total)
    act = g.make_activation(m, ks, c_total, ctx)
    halo = max(len(ks.angular) // 2, 1)
    full = g.init_uniform(m, c_total, ctx)
    shards = [_shard(ctx, m, c_total, *partition(c_total, G, r), halo) for r in range(G)]
    plans = [halo_plan(c_total, G, r, halo) for r in range(G)]

    def exchange():
        for r, t in enumerate(shards):
            pl = plans[r]
            left, right = shards[pl.left], shards[pl.right]
            lp, rp = plans[pl.left], plans[pl.right]
            check(ctx.lib.gl_tensor_copy_planes(ctx.h, t.h, pl.recv_left[0], left.h, lp.send_right[0], halo))
            check(ctx.lib.gl_tensor_copy_planes(ctx.h, t.h, pl.recv_right[0], right.h, rp.send_left[0], halo))
        ctx.synchronize()

    def step_all(u, v, w):
        g.step(full, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        for t in shards:
            g.step_async(t, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        ctx.synchronize()
        _emulate_max_allreduce(ctx, shards)
        for t in shards:
            check(ctx.lib.gl_shard_finalize(ctx.h, t.h))
        exchange()

    rng = Rng(G + c_total)
    for _ in range(4):
        step_all(*random_motion(rng))
    js, is_ = np.nonzero(occ == 0)
    q = len(is_) // 3
    a, r = simple_scan(occ, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.4)
    scan = g.LidarScan(a, r, 8.0)
    params = g.LikelihoodParams()
    for obs in range(2):
        ref_s = g.dither_samples(full, 512)
        g.observation_update(full, ref_s, scan, m, f, params)
        planes = []
        for t in shards:
            pl = torch.empty(128 * 96, dtype=torch.float64, device="cuda")
            check(ctx.lib.gl_shard_belief_map(ctx.h, t.h, C.c_void_p(pl.data_ptr())))
            planes.append(pl)
        ctx.synchronize()
        red = torch.stack(planes).max(dim=0).values.contiguous()
        torch.cuda.synchronize()
        cap = 4 * 512 + 64
        cells = np.zeros(2 * cap, np.int32)
        n, mass = C.c_int(), C.c_double()
        check(ctx.lib.gl_dither_device(ctx.h, C.c_void_p(red.data_ptr()), 128, 96, 512,
                                       cells.ctypes.data_as(C.POINTER(C.c_int)), cap, C.byref(n), C.byref(mass)))
        cells = cells[: 2 * n.value]
        assert np.array_equal(cells.reshape(-1, 2), ref_s.cells), f"obs {obs}: samples differ"
        assert np.float64(mass.value).tobytes() == np.float64(ref_s.source_mass).tobytes()
        assert n.value > 0
        aa = np.ascontiguousarray(a, dtype=np.float64)
        rr = np.ascontiguousarray(r, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        for t in shards:
            check(ctx.lib.gl_shard_observe(ctx.h, t.h, cells.ctypes.data_as(C.POINTER(C.c_int)), n.value,
                                           aa.ctypes.data_as(dp), rr.ctypes.data_as(dp), aa.size, 8.0, m.h, f.h,
                                           g.gridloc._lp(params)))
        ctx.synchronize()
        _emulate_max_allreduce(ctx, shards)
        for t in shards:
            check(ctx.lib.gl_shard_observe_finalize(ctx.h, t.h))
        exchange()
        if obs == 0:  # download materialises the pending 1/max rescale ...
            got = np.concatenate([t.values() for t in shards], axis=0)
            assert_bitwise(got, full.values(), f"G={G} observation {obs}")
        step_all(0.1, 0.0, 0.0)  # ... else the next step's kernel applies it
        got = np.concatenate([t.values() for t in shards], axis=0)
        assert_bitwise(got, full.values(), f"G={G} step after observation {obs}")


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_theta_shard_observe_world1(ctx, exchange):
    """ThetaShard.observe (the sharded Localizer::observe glue over
    observe_collectives) at world size 1: samples and tensor bitwise the
    unsharded dither_samples + observation_update, then a step."""
    from paper_1910_00572_b200.floorplan import simple_scan
    from paper_1910_00572_b200.sharding import ThetaShard
    occ = make_floorplan(96, 64, seed=5)
    m = g.OccupancyMap(96, 64, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    C_ = 72
    ks = g.build_kernels(g.MotionNoise(), C_, 0.1, 2 * math.pi / C_)
    act = g.make_activation(m, ks, C_, ctx)
    full = g.init_uniform(m, C_, ctx)
    sh = ThetaShard(m, C_, 1, 0, 1, ctx, exchange=exchange)
    try:
        rng = Rng(9)
        js, is_ = np.nonzero(occ == 0)
        a, r = simple_scan(occ, is_[10] * 0.1 + 0.05, js[10] * 0.1 + 0.05, 0.2)
        scan = g.LidarScan(a, r, 8.0)
        for it in range(3):
            u = g.OdometryDelta(*random_motion(rng))
            g.step(full, u, m, ks, act, ctx)
            sh.step(u, ks, act)
            ref_s = g.dither_samples(full, 256)
            g.observation_update(full, ref_s, scan, m, f)
            s = sh.observe(scan, f, budget=256)
            assert np.array_equal(s.cells, ref_s.cells) and s.source_mass == ref_s.source_mass
            ctx.synchronize()
            assert_bitwise(sh.t.values(), full.values(), f"{exchange} observe {it}")
    finally:
        sh.close()
