"""theta-slab sharding of one belief tensor across ranks.

Rank r of G owns global channels [r*C/G, (r+1)*C/G). The step is channel-
local except the circular angular stencil (+-H channels,
belief_tensor.cpp:449-451), so each rank stores `halo` neighbour planes per
side and a step is

  1. the fused kernel on the local slab (reads halo planes, writes interior
     planes, leaves the local max),
  2. an all-reduce MAX of the 8-byte max (uint64 bits of a double >= 0: the
     integer order is the value order),
  3. finalize (extinguish status, pending 1/max rescale — global, so every
     rank scales identically),
  4. the halo exchange: my first/last `halo` interior planes go to the
     left/right neighbour's upper/lower halo.

The exchange has two forms. "peer" (default): the fused step kernel reads
its halo input planes straight from the neighbours' buffers through peer
memory (CUDA IPC mappings, TMA over NVLink P2P; gl_shard_set_peers), so the
transfer overlaps the compute tile by tile and there is no exchange step at
all; the MAX all-reduce that follows every step is the barrier that orders
a neighbour's writes of a buffer before these reads, and these reads before
the neighbour overwrites it. "nccl": NCCL send/recv of the planes after the
step (the north star's form; kept for fabrics without P2P).

No per-element operation changes, so the sharded belief is bitwise the
unsharded one. The exchange plan and the argmax combine are pure functions
(tested with gloo on CPU); device memory is handed to torch.distributed
through __cuda_array_interface__ (zero copy) on the library's own stream.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check


def partition(c_total: int, world: int, rank: int):
    """[c_begin, c_end) of rank (contiguous, sizes differ by at most 1)."""
    return rank * c_total // world, (rank + 1) * c_total // world


@dataclass(frozen=True)
class HaloPlan:
    """Storage-plane ranges for one rank's halo exchange.

    storage plane q <-> global channel (c_begin - halo + q) mod c_total."""
    rank: int
    world: int
    left: int           # rank owning the channels just below mine (circular)
    right: int          # rank owning the channels just above mine
    send_left: tuple    # (q0, count): my first `halo` interior planes
    send_right: tuple   # my last `halo` interior planes
    recv_left: tuple    # my lower halo planes (from the left neighbour's last)
    recv_right: tuple   # my upper halo planes (from the right neighbour's first)


def halo_plan(c_total: int, world: int, rank: int, halo: int) -> HaloPlan:
    c0, c1 = partition(c_total, world, rank)
    n = c1 - c0
    if halo > min(partition(c_total, world, r)[1] - partition(c_total, world, r)[0] for r in range(world)):
        raise ValueError("halo wider than a shard: use fewer ranks or a larger channel count")
    return HaloPlan(rank, world, (rank - 1) % world, (rank + 1) % world,
                    send_left=(halo, halo), send_right=(n, halo),
                    recv_left=(0, halo), recv_right=(halo + n, halo))


@dataclass(frozen=True)
class PeerPlan:
    """Where the fused step reads this rank's halo input planes (peer mode):
    storage plane s < halo comes from rank lo_rank's storage plane
    s + lo_count (lo_count = its interior channel count), plane s >= halo + n
    from rank hi_rank's plane s - n."""
    lo_rank: int
    lo_count: int
    hi_rank: int
    hi_count: int


def peer_plan(c_total: int, world: int, rank: int, halo: int) -> PeerPlan:
    left, right = (rank - 1) % world, (rank + 1) % world
    lc0, lc1 = partition(c_total, world, left)
    rc0, rc1 = partition(c_total, world, right)
    halo_plan(c_total, world, rank, halo)  # validates halo against the shard sizes
    return PeerPlan(left, lc1 - lc0, right, rc1 - rc0)


def exchange_ipc_handles(dist, mine, group=None):
    """All-gather every rank's (buffer-0, buffer-1) IPC handles (bytes)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, tuple(bytes(h) for h in mine), group=group)
    return out


def combine_argmax(cands):
    """cands: per-rank (value, global flat index); the reference keeps the
    first strict maximum in (k, j, i) order (belief_tensor.cpp:518-527), i.e.
    the largest value with the lowest flat index."""
    best = None
    for v, idx in cands:
        if not (v > -1.0):
            continue
        if best is None or v > best[0] or (v == best[0] and idx < best[1]):
            best = (v, idx)
    return best


def exchange_planes(dist, planes, plan: HaloPlan, group=None):
    """Halo exchange through torch.distributed point-to-point ops.
    planes(q0, count) returns a tensor view of storage planes q0..q0+count-1
    (a zero-copy device alias on GPUs, a CPU tensor under gloo in tests)."""
    # Messages between one pair of ranks match in issue order (NCCL has no
    # tags), and with two ranks left == right: every rank sends right-edge
    # then left-edge and receives lower-halo then upper-halo, so the first
    # message a rank gets from its left neighbour is that neighbour's right
    # edge, the second from its right neighbour is that neighbour's left edge.
    ops = [
        dist.P2POp(dist.isend, planes(*plan.send_right), plan.right, group),
        dist.P2POp(dist.isend, planes(*plan.send_left), plan.left, group),
        dist.P2POp(dist.irecv, planes(*plan.recv_left), plan.left, group),
        dist.P2POp(dist.irecv, planes(*plan.recv_right), plan.right, group),
    ]
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def observe_collectives(dist, group, rank: int, world: int, root: int, plane, max_bits, local_map, dither,
                        apply, finalize):
    """The collective skeleton of a sharded observation,
    device work injected as callables so the host logic runs under gloo too:
      local_map(plane)       this rank's per-cell max into `plane` (float64)
      dither(plane) -> (cells int32 (n, 2), mass)   called on `root` only
      apply(cells, n)        likelihoods over all channels, own channels
                             multiplied, local max into `max_bits`
      finalize()             the 1/max rescale and status
    Returns (cells, mass), identical on every rank."""
    import numpy as np
    import torch
    local_map(plane)
    if world > 1:
        dist.all_reduce(plane, op=dist.ReduceOp.MAX, group=group)
    hdr = torch.zeros(2, dtype=torch.float64, device=plane.device)  # n, source mass
    cells = None
    if rank == root:
        cells, mass = dither(plane)
        hdr[0], hdr[1] = float(len(cells)), float(mass)
    if world > 1:
        dist.broadcast(hdr, src=root, group=group)
    n, mass = int(hdr[0].item()), float(hdr[1].item())
    buf = torch.zeros(max(2 * n, 2), dtype=torch.int32, device=plane.device)
    if rank == root and n:
        buf[: 2 * n] = torch.from_numpy(np.ascontiguousarray(cells, dtype=np.int32).reshape(-1)).to(plane.device)
    if world > 1:
        dist.broadcast(buf, src=root, group=group)
    cells = np.ascontiguousarray(buf[: 2 * n].cpu().numpy(), dtype=np.int32).reshape(-1, 2)
    if n == 0:  # observation.cpp:117: an empty sample set is a no-op
        return cells, mass
    apply(cells, n)
    if world > 1:
        dist.all_reduce(max_bits, op=dist.ReduceOp.MAX, group=group)
    finalize()
    return cells, mass


class _CAI:
    """Zero-copy device view for torch.as_tensor(..., device='cuda')."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


class ThetaShard:
    """This rank's slab. Collectives go through torch.distributed (NCCL) on
    the library's stream; one process per GPU."""

    def __init__(self, m, c_total: int, halo: int, rank: int, world: int, ctx, group=None,
                 exchange: str = "peer"):
        import torch
        import torch.distributed as dist
        from .gridloc import BeliefTensor
        self.torch, self.dist, self.group = torch, dist, group
        self.ctx, self.map = ctx, m
        self.c_total, self.halo, self.rank, self.world = c_total, halo, rank, world
        self.c_begin, self.c_end = partition(c_total, world, rank)
        self.plan = halo_plan(c_total, world, rank, halo)
        h = C.c_void_p()
        check(ctx.lib.gl_shard_init_uniform(ctx.h, m.h, c_total, self.c_begin, self.c_end, halo, C.byref(h)))
        self.t = BeliefTensor(ctx=ctx, _handle=h)
        self.stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", ctx.device))
        self.plane_elems = m.width() * m.height()
        if exchange not in ("peer", "nccl"):
            raise ValueError("exchange must be 'peer' or 'nccl'")
        self.exchange = exchange
        self._ipc_open = []
        if exchange == "peer":
            self._set_peers()

    def _buffer_base(self, t_handle, buf):
        p = C.POINTER(C.c_double)()
        check(self.ctx.lib.gl_tensor_buffer_ptr(self.ctx.h, t_handle, buf, 0, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    def _set_peers(self):
        """Point the fused step's halo reads at the neighbours' buffers: this
        process's own buffers when world == 1, CUDA IPC mappings of the
        neighbours' buffers otherwise."""
        lib, pp = self.ctx.lib, peer_plan(self.c_total, self.world, self.rank, self.halo)
        if self.world == 1:
            bases = {self.rank: [self._buffer_base(self.t.h, b) for b in (0, 1)]}
        else:
            mine = []
            for b in (0, 1):
                h = (C.c_ubyte * 64)()
                check(lib.gl_ipc_get_handle(self.ctx.h, self.t.h, b, h))
                mine.append(bytes(h))
            allh = exchange_ipc_handles(self.dist, mine, self.group)
            bases = {}
            for r in {pp.lo_rank, pp.hi_rank}:
                bases[r] = []
                for b in (0, 1):
                    buf = (C.c_ubyte * 64).from_buffer_copy(allh[r][b])
                    ptr = C.c_void_p()
                    check(lib.gl_ipc_open(self.ctx.h, buf, C.byref(ptr)))
                    self._ipc_open.append(ptr.value)
                    bases[r].append(ptr.value)
        lo, hi = bases[pp.lo_rank], bases[pp.hi_rank]
        check(lib.gl_shard_set_peers(self.ctx.h, self.t.h, C.c_void_p(lo[0]), C.c_void_p(lo[1]), pp.lo_count,
                                     C.c_void_p(hi[0]), C.c_void_p(hi[1]), pp.hi_count))

    def close(self):
        """Unmap the neighbours' IPC buffers (peer mode, world > 1)."""
        for ptr in self._ipc_open:
            check(self.ctx.lib.gl_ipc_close(self.ctx.h, C.c_void_p(ptr)))
        self._ipc_open = []

    def _planes(self, q0: int, count: int):
        p = C.POINTER(C.c_double)()
        check(self.ctx.lib.gl_tensor_plane_ptr(self.ctx.h, self.t.h, q0, C.byref(p)))
        ptr = C.cast(p, C.c_void_p).value
        return self.torch.as_tensor(_CAI(ptr, (count, self.plane_elems), "<f8"), device=f"cuda:{self.ctx.device}")

    def _max_tensor(self):
        p = C.POINTER(C.c_uint64)()
        check(self.ctx.lib.gl_tensor_max_ptr(self.ctx.h, self.t.h, C.byref(p)))
        return self.torch.as_tensor(_CAI(C.cast(p, C.c_void_p).value, (1,), "<i8"),
                                    device=f"cuda:{self.ctx.device}")

    def step(self, u, kernels, act):
        """One sharded Algorithm-1 step (asynchronous on the device)."""
        from .gridloc import step_async
        step_async(self.t, u, self.map, kernels, act, self.ctx)
        with self.torch.cuda.stream(self.stream):
            if self.world > 1:
                self.dist.all_reduce(self._max_tensor(), op=self.dist.ReduceOp.MAX, group=self.group)
            check(self.ctx.lib.gl_shard_finalize(self.ctx.h, self.t.h))
            if self.exchange == "nccl":
                self.exchange_halos()

    def exchange_halos(self):
        """Explicit exchange of the current buffer's edge planes (the "nccl"
        mode's per-step exchange; peer mode never needs it)."""
        pl = self.plan
        if self.world == 1:
            lib = self.ctx.lib
            # circular: lower halo <- my last planes, upper halo <- my first
            check(lib.gl_tensor_copy_planes(self.ctx.h, self.t.h, pl.recv_left[0], self.t.h, pl.send_right[0],
                                            self.halo))
            check(lib.gl_tensor_copy_planes(self.ctx.h, self.t.h, pl.recv_right[0], self.t.h, pl.send_left[0],
                                            self.halo))
            return
        exchange_planes(self.dist, self._planes, pl, self.group)

    def status(self):
        from .gridloc import tensor_status
        tensor_status(self.t)

    def observe(self, scan, field, params=None, budget: int = 512, root: int = 0):
        """Sharded Localizer::observe (localizer.cpp:48-59): the global
        belief_map as a MAX all-reduce of the shards' local maps, dither on
        `root`, the samples broadcast, every rank's likelihoods over all
        channels (identical sequential mean), its own channels multiplied,
        the max all-reduced and the 1/max rescale finalised
        (observe_collectives). Returns the SampleSet (same on every rank)."""
        import numpy as np
        from .gridloc import LikelihoodParams, SampleSet, _d, _i, _lp
        torch, lib, ctx = self.torch, self.ctx.lib, self.ctx
        params = params or LikelihoodParams()
        W, H = self.map.width(), self.map.height()
        cap = max(1, min(W * H, 4 * max(budget, 1) + 64))
        a = np.ascontiguousarray(scan.angles, dtype=np.float64)
        r = np.ascontiguousarray(scan.ranges, dtype=np.float64)

        def local_map(plane):
            check(lib.gl_shard_belief_map(ctx.h, self.t.h, C.c_void_p(plane.data_ptr())))

        def dither(plane):
            cells = np.zeros(2 * cap, np.int32)
            n, mass = C.c_int(), C.c_double()
            check(lib.gl_dither_device(ctx.h, C.c_void_p(plane.data_ptr()), W, H, budget, _i(cells), cap,
                                       C.byref(n), C.byref(mass)))
            return cells[: 2 * n.value].reshape(-1, 2), mass.value

        def apply(cells, n):
            flat = np.ascontiguousarray(cells, dtype=np.int32).reshape(-1)
            check(lib.gl_shard_observe(ctx.h, self.t.h, _i(flat), n, _d(a), _d(r), a.size, scan.max_range,
                                       self.map.h, field.h, _lp(params)))

        def finalize():
            check(lib.gl_shard_observe_finalize(ctx.h, self.t.h))
            if self.exchange == "nccl":
                self.exchange_halos()

        with torch.cuda.stream(self.stream):
            plane = torch.empty(W * H, dtype=torch.float64, device=f"cuda:{ctx.device}")
            cells, mass = observe_collectives(self.dist, self.group, self.rank, self.world, root, plane,
                                              self._max_tensor(), local_map, dither, apply, finalize)
        return SampleSet(cells.copy(), mass)

    def argmax(self):
        """Global argmax_state: local candidate, all-gather, lowest-index rule."""
        from .gridloc import BeliefExtinguishedError, argmax_state
        W = self.map.width()
        try:
            e = argmax_state(self.t)
            flat = (self.c_begin + e.k) * self.plane_elems + e.j * W + e.i
            val = self.t.at(e.i, e.j, e.k)
        except BeliefExtinguishedError:
            val, flat = -1.0, 0
        t = self.torch.tensor([val, float(flat)], dtype=self.torch.float64, device=f"cuda:{self.ctx.device}")
        out = [self.torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        best = combine_argmax([(float(o[0]), int(o[1])) for o in out])
        if best is None:
            raise RuntimeError("argmax on an all-zero belief tensor")
        plane = self.plane_elems
        k, p = divmod(best[1], plane)
        j, i = divmod(p, self.map.width())
        return best[0], (i, j, k)
