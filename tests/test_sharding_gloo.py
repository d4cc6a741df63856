"""Multi-rank host logic of the theta-slab sharding, world size 2 and 3 with
the gloo backend on CPU (one process per rank, 127.0.0.1 rendezvous):
partitioning, the halo plan, the point-to-point exchange of storage planes,
the MAX all-reduce on the uint64 bits of the step max, and the argmax
combine rule. Device compute is covered by tests/test_gpu_sharding.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_00572_b200.sharding import (combine_argmax, exchange_ipc_handles, exchange_planes, halo_plan,
                                            partition, peer_plan)

PLANE = 12  # elements per plane in these host-only tests


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, c_total, halo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c0, c1 = partition(c_total, world, rank)
        n = c1 - c0
        plan = halo_plan(c_total, world, rank, halo)
        # storage: halo | interior | halo; interior plane of channel k holds k
        store = torch.full((n + 2 * halo, PLANE), -1.0, dtype=torch.float64)
        for qq in range(halo, halo + n):
            store[qq] = float(c0 + qq - halo)

        exchange_planes(dist, lambda q0, cnt: store[q0:q0 + cnt], plan)
        got = [float(store[qq, 0]) for qq in range(n + 2 * halo)]
        want = [float((c0 - halo + qq) % c_total) for qq in range(n + 2 * halo)]

        # MAX all-reduce of the step max as uint64 bits of doubles >= 0
        local = np.array([0.25 * (rank + 1)], dtype=np.float64).view(np.int64)
        t = torch.from_numpy(local.copy())
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gmax = float(t.numpy().view(np.float64)[0])

        # argmax combine: ties across ranks resolve to the lowest flat index
        cand = torch.tensor([1.0, float(1000 - rank)], dtype=torch.float64)
        outs = [torch.zeros_like(cand) for _ in range(world)]
        dist.all_gather(outs, cand)
        best = combine_argmax([(float(o[0]), int(o[1])) for o in outs])
        # peer mode: every rank learns every rank's two IPC handles
        mine = (bytes([rank]) * 64, bytes([rank + 100]) * 64)
        allh = exchange_ipc_handles(dist, mine)
        ipc_ok = all(allh[r] == (bytes([r]) * 64, bytes([r + 100]) * 64) for r in range(world))
        q.put((rank, got == want and ipc_ok, got, want, gmax, best))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,c_total,halo", [(2, 8, 1), (3, 36, 1), (2, 360, 3), (3, 16, 2)])
def test_halo_exchange_allreduce_argmax(world, c_total, halo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, c_total, halo, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, got, want, gmax, best in res:
        assert ok, (rank, got, want)
        assert gmax == 0.25 * world
        assert best == (1.0, 1000 - (world - 1))


def test_partition_and_plan():
    assert [partition(72, 8, r) for r in range(8)] == [(9 * r, 9 * r + 9) for r in range(8)]
    assert sum(b - a for a, b in (partition(10, 3, r) for r in range(3))) == 10
    p = halo_plan(360, 8, 0, 3)
    assert (p.left, p.right) == (7, 1)
    assert p.send_left == (3, 3) and p.send_right == (45, 3)
    assert p.recv_left == (0, 3) and p.recv_right == (48, 3)
    with pytest.raises(ValueError):
        halo_plan(8, 8, 0, 2)


def test_combine_argmax_rules():
    assert combine_argmax([(0.5, 10), (0.7, 99), (0.7, 3)]) == (0.7, 3)
    assert combine_argmax([(-1.0, 0), (-1.0, 5)]) is None
    assert combine_argmax([(float("nan"), 0), (0.1, 4)]) == (0.1, 4)


@pytest.mark.parametrize("world,c_total,halo", [(1, 72, 1), (2, 8, 1), (3, 36, 1), (8, 360, 3), (3, 16, 2),
                                                (5, 72, 1)])
def test_peer_plan_reads_the_channels_the_halo_holds(world, c_total, halo):
    """Peer mode reads halo input planes from the neighbours' buffers: own
    storage plane s < halo from the left neighbour's plane s + lo_count,
    s >= halo + n from the right neighbour's plane s - n. Those planes must
    hold exactly the channels the own halo planes stand for (storage plane q
    of rank r holds channel (c_begin_r - halo + q) mod C), and must be
    interior planes of the neighbour (it wrote them in the last step)."""
    for r in range(world):
        pp = peer_plan(c_total, world, r, halo)
        pl = halo_plan(c_total, world, r, halo)
        assert (pp.lo_rank, pp.hi_rank) == (pl.left, pl.right)
        c0, c1 = partition(c_total, world, r)
        n = c1 - c0
        lc0, lc1 = partition(c_total, world, pl.left)
        rc0, rc1 = partition(c_total, world, pl.right)
        assert (pp.lo_count, pp.hi_count) == (lc1 - lc0, rc1 - rc0)
        for s in range(halo):
            q = s + pp.lo_count
            assert halo <= q < halo + pp.lo_count
            assert (lc0 - halo + q) % c_total == (c0 - halo + s) % c_total
        for s in range(halo + n, 2 * halo + n):
            q = s - n
            assert halo <= q < halo + pp.hi_count
            assert (rc0 - halo + q) % c_total == (c0 - halo + s) % c_total


def _obs_worker(rank, world, port, q, empty):
    from paper_1910_00572_b200.sharding import observe_collectives
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(rank)
        mine = rng.random(PLANE)                      # this rank's local belief map
        calls = {"dither": 0, "apply": None, "finalize": 0}
        plane = torch.zeros(PLANE, dtype=torch.float64)
        max_bits = torch.from_numpy(np.array([0.0], np.float64).view(np.int64).copy())

        def local_map(p):
            p.copy_(torch.from_numpy(mine))

        def dither(p):
            calls["dither"] += 1
            if empty:
                return np.zeros((0, 2), np.int32), 0.0
            v = p.numpy()
            idx = np.argsort(-v)[:3]                   # deterministic "samples" from the reduced map
            return np.stack([idx, idx + 100], axis=1).astype(np.int32), float(v.sum())

        def apply(cells, n):
            calls["apply"] = (cells.copy(), n)
            max_bits.copy_(torch.from_numpy(np.array([0.5 + rank], np.float64).view(np.int64)))

        def finalize():
            calls["finalize"] += 1

        cells, mass = observe_collectives(dist, None, rank, world, 0, plane, max_bits, local_map, dither, apply,
                                          finalize)
        gmax = float(max_bits.numpy().view(np.float64)[0])
        q.put((rank, plane.numpy().copy(), cells, mass, calls["dither"], calls["apply"], calls["finalize"], gmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,empty", [(2, False), (3, False), (2, True)])
def test_observation_collectives(world, empty):
    """Sharded observation skeleton: the belief map is the elementwise MAX
    of the ranks' local maps, only the root dithers, every rank gets the
    root's samples and mass, the step max is MAX-reduced before finalize,
    and an empty sample set skips apply/finalize everywhere."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_obs_worker, args=(r, world, port, q, empty)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.max([np.random.default_rng(r).random(PLANE) for r in range(world)], axis=0)
    root_cells, root_mass = res[0][2], res[0][3]
    for rank, plane, cells, mass, nd, applied, nfin, gmax in res:
        assert np.array_equal(plane, want)
        assert np.array_equal(cells, root_cells) and mass == root_mass
        assert nd == (1 if rank == 0 else 0)
        if empty:
            assert len(cells) == 0 and applied is None and nfin == 0
        else:
            assert len(cells) == 3 and np.array_equal(applied[0], root_cells) and applied[1] == 3
            assert nfin == 1 and gmax == 0.5 + (world - 1)
