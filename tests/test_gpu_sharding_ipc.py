"""The cross-process theta-sharded path end to end on ONE GPU: two processes
(one per shard, as on a multi-GPU box), each with its own context, its
neighbour's ping-pong buffers mapped through CUDA IPC (gl_ipc_get_handle /
gl_ipc_open) so the fused step's TMA reads its halo input planes straight
from the other process's memory, and the 8-byte step-max all-reduce plus the
observation collectives over gloo (NCCL refuses two ranks on one device).
The kernels never wait on each other: every cross-process ordering is the
host-side all-reduce (sharding.py). ThetaShard.step / observe / argmax must
be bitwise the unsharded tensor (sharding changes no
per-element operation)."""
import math
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W, H, STEPS = 128, 96, 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _motions():
    from tests.helpers import Rng, random_motion
    rng = Rng(77)
    return [random_motion(rng) for _ in range(STEPS)] + [(0.1, 0.0, 0.0)]


def _scan(occ):
    from paper_1910_00572_b200.floorplan import simple_scan
    js, is_ = np.nonzero(occ == 0)
    q = len(is_) // 2
    return simple_scan(occ, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.4)


def _worker(rank, world, port, c_total, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import paper_1910_00572_b200 as g
    from paper_1910_00572_b200.sharding import ThetaShard
    from tests.helpers import make_floorplan
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = g.Context(0)
        occ = make_floorplan(W, H, seed=41)
        m = g.OccupancyMap(W, H, 0.1, occ, ctx=ctx)
        f = g.DistanceField(m, ctx)
        ks = g.build_kernels(g.MotionNoise(), c_total, 0.1, 2 * math.pi / c_total)
        act = g.make_activation(m, ks, c_total, ctx)
        halo = max(1, len(ks.angular) // 2)
        shard = ThetaShard(m, c_total, halo, rank, world, ctx, exchange="peer")
        assert shard._ipc_open, "peer mode across processes must map the neighbours' buffers over CUDA IPC"
        for (u, v, w) in _motions()[:4]:
            shard.step(g.OdometryDelta(u, v, w), ks, act)
        a, r = _scan(occ)
        smp = shard.observe(g.LidarScan(a, r, 8.0), f)
        for (u, v, w) in _motions()[4:]:
            shard.step(g.OdometryDelta(u, v, w), ks, act)
        ctx.synchronize()
        shard.status()
        val, ijk = shard.argmax()
        np.save(os.path.join(outdir, f"rank{rank}.npy"), shard.t.values())
        np.save(os.path.join(outdir, f"samples{rank}.npy"), smp.cells)
        with open(os.path.join(outdir, f"meta{rank}.txt"), "w") as fh:
            fh.write(f"{shard.c_begin} {shard.c_end} {smp.source_mass!r} {val!r} {ijk[0]} {ijk[1]} {ijk[2]} "
                     f"{shard.t.theta_t()!r}\n")
        dist.barrier()  # neighbours stop reading my buffers before I free them
        shard.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("c_total", [72, 360])
def test_two_process_ipc_shards_bitwise_equal_unsharded(ctx, c_total):
    import torch.multiprocessing as mp
    import paper_1910_00572_b200 as g
    from tests.helpers import assert_bitwise, make_floorplan
    world = 2
    with tempfile.TemporaryDirectory() as outdir:
        mpc = mp.get_context("spawn")
        port = _free_port()
        procs = [mpc.Process(target=_worker, args=(r, world, port, c_total, outdir)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
            assert p.exitcode == 0, f"shard process exit code {p.exitcode}"
        # the unsharded reference run in this process
        occ = make_floorplan(W, H, seed=41)
        m = g.OccupancyMap(W, H, 0.1, occ, ctx=ctx)
        f = g.DistanceField(m, ctx)
        ks = g.build_kernels(g.MotionNoise(), c_total, 0.1, 2 * math.pi / c_total)
        act = g.make_activation(m, ks, c_total, ctx)
        t = g.init_uniform(m, c_total, ctx)
        for (u, v, w) in _motions()[:4]:
            g.step(t, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        a, r = _scan(occ)
        smp = g.dither_samples(t, 512)
        g.observation_update(t, smp, g.LidarScan(a, r, 8.0), m, f, g.LikelihoodParams())
        for (u, v, w) in _motions()[4:]:
            g.step(t, g.OdometryDelta(u, v, w), m, ks, act, ctx)
        full = t.values()
        est = g.argmax_state(t)
        for rank in range(world):
            meta = open(os.path.join(outdir, f"meta{rank}.txt")).read().split()
            c0, c1 = int(meta[0]), int(meta[1])
            assert_bitwise(np.load(os.path.join(outdir, f"rank{rank}.npy")), full[c0:c1], f"rank {rank} slab")
            assert np.array_equal(np.load(os.path.join(outdir, f"samples{rank}.npy")), smp.cells)
            assert float(meta[2]) == smp.source_mass
            assert (int(meta[4]), int(meta[5]), int(meta[6])) == (est.i, est.j, est.k)
            assert float(meta[7]) == t.theta_t()
