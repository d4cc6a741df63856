"""GPU parity of the Algorithm-1 step (belief_tensor.cpp:396-498) against the
CPU oracle, bit-exact in FP64 (the bar for this path). Both the fused sm_100a
kernel and the generic kernel chain are checked; inputs follow the
reference's own step tests (proj/tests/test_belief_engine.cpp:203-449)."""
import math

import numpy as np
import pytest

import paper_1910_00572_b200 as g
from paper_1910_00572_b200._lib import GL_PATH_AUTO, GL_PATH_FUSED, GL_PATH_GENERIC
from tests.helpers import (Rng, assert_bitwise, make_empty_room, make_floorplan, random_map, random_motion,
                           random_tensor, twin_room_map)

pytestmark = pytest.mark.gpu


def _setup(ctx, occ, channels, noise, res=0.1):
    h, w = occ.shape
    m = g.OccupancyMap(w, h, res, occ, ctx=ctx)
    dth = 2.0 * math.pi / channels
    ks = g.build_kernels(g.MotionNoise(*noise), channels, res, dth)
    act = g.make_activation(m, ks, channels, ctx)
    return m, ks, act


def _run_pair(ctx, port, occ, channels, noise, motions, path, B0=None, res=0.1, check_every=True):
    """Run the same motions on the GPU and the oracle; compare bitwise."""
    ctx.set_path(path)
    try:
        m, ks, act = _setup(ctx, occ, channels, noise, res)
        cells = m.cells()
        pks = port.build_kernels(*noise, channels, res)
        _, pinv = port.make_activation(cells, pks, channels)
        if B0 is None:
            t = g.init_uniform(m, channels, ctx)
            B = port.init_uniform(cells, channels)
        else:
            h, w = occ.shape
            t = g.BeliefTensor(w, h, channels, res, ctx=ctx)
            t.set_values(B0)
            B = np.array(B0, dtype=np.float64, copy=True)
        th = 0.0
        for s, (u, v, w_) in enumerate(motions):
            rc, th = port.step(B, th, u, v, w_, cells, res, pks, pinv)
            if rc:
                with pytest.raises(g.BeliefExtinguishedError):
                    g.step(t, g.OdometryDelta(u, v, w_), m, ks, act, ctx)
            else:
                g.step(t, g.OdometryDelta(u, v, w_), m, ks, act, ctx)
            assert t.theta_t() == th
            if check_every or s == len(motions) - 1:
                assert_bitwise(t.values(), B, f"step {s} path {path}")
        return t, B
    finally:
        ctx.set_path(GL_PATH_AUTO)


CASES = [
    # (map builder, channels, noise)  -- default noise at several channel counts
    ("floor96x80", 72, (0.03, 0.03, 0.012)),    # separable r=1, 3 angular taps
    ("floor96x80", 36, (0.03, 0.03, 0.012)),    # angular degenerate (1 tap)
    ("floor96x80", 360, (0.03, 0.03, 0.012)),   # 7 angular taps (h = 3)
    ("random28x22", 8, (0.06, 0.05, 0.05)),     # anisotropic r=2 dense (generic)
    ("random16x16", 8, (0.06, 0.05, 0.07)),     # the reference's oracle test inputs
    ("empty40x40", 8, (0.06, 0.06, 0.08)),      # isotropic r=2, h=1
    ("twin", 8, (0.05, 0.05, 2.0)),             # folded angular kernel (generic)
    ("random37x29", 16, (0.03, 0.03, 0.012)),   # odd width: TMA needs even W -> generic
    ("floor130x70", 72, (0.2, 0.2, 0.012)),     # isotropic r=6 (generic separable)
    ("random40x32", 12, (0.3, 0.2, 0.1)),       # anisotropic r=9: convolve_plane's generic interior order
]


def _map(name):
    if name == "floor96x80":
        return make_floorplan(96, 80, seed=3)
    if name == "floor130x70":
        return make_floorplan(130, 70, seed=4)
    if name == "random28x22":
        return random_map(28, 22, 0.12, 55)
    if name == "random16x16":
        return random_map(16, 16, 0.15, 42)
    if name == "random40x32":
        return random_map(40, 32, 0.1, 91)
    if name == "random37x29":
        return random_map(37, 29, 0.15, 7)
    if name == "empty40x40":
        return make_empty_room(40, 40)
    if name == "twin":
        return twin_room_map()
    raise KeyError(name)


@pytest.mark.parametrize("name,channels,noise", CASES)
@pytest.mark.parametrize("path", [GL_PATH_AUTO, GL_PATH_GENERIC])
def test_step_bit_exact_random_motions(ctx, port, name, channels, noise, path):
    occ = _map(name)
    rng = Rng(7)
    motions = [random_motion(rng) for _ in range(6)]
    motions += [(0.1, 0.0, 0.0), (0.0, 0.0, 0.0), (0.3, -0.2, 0.0), (-1.7, 2.4, 1.1)]
    _run_pair(ctx, port, occ, channels, noise, motions, path)


@pytest.mark.parametrize("channels", [72, 36])
def test_rotation_only_slot_bit_exact(ctx, port, channels):
    """Localizer's rotation-only kernels (localizer.cpp:16-20): r = 0."""
    occ = make_floorplan(128, 96, seed=5)
    rng = Rng(11)
    motions = [(0.0, 0.0, rng.uniform(-0.1, 0.1)) for _ in range(5)] + [(0.02, 0.01, 0.05)]
    _run_pair(ctx, port, occ, channels, (1e-4, 1e-4, 0.012), motions, GL_PATH_FUSED)


def test_fused_path_is_used_for_default_kernels(ctx, port):
    """Forcing GL_PATH_FUSED must succeed for the Localizer's kernel sets."""
    occ = make_floorplan(64, 64, seed=1)
    _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), [(0.1, 0.0, 0.0), (0.05, 0.02, 0.03)], GL_PATH_FUSED)


def test_fused_tile_edges_bit_exact(ctx, port):
    """Grid sizes that are not multiples of the 64 x ROWS tile."""
    for (w, h) in [(66, 17), (130, 35), (64, 16), (200, 3)]:
        occ = random_map(w, h, 0.1, w * 31 + h)
        rng = Rng(w)
        B0 = random_tensor(occ, 72, seed=w + h, free_only=False)
        motions = [random_motion(rng, 0.3, 0.3, 0.2) for _ in range(3)]
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED, B0=B0)


@pytest.mark.parametrize("fast", [True, False])
@pytest.mark.parametrize("w,h,channels", [(37, 29, 72), (129, 35, 72), (3, 40, 36), (255, 17, 360), (5, 9, 8)])
def test_fused_odd_widths_bit_exact(ctx, port, fast, w, h, channels):
    """Odd W: 8*W bytes is not a TMA row stride, so the fused kernel loads
    its boxes with per-lane cp.async copies (zero-filled outside the grid)
    instead of one TMA box — same smem layout and arithmetic."""
    occ = random_map(w, h, 0.12, w * 7 + h)
    rng = Rng(w + h)
    B0 = random_tensor(occ, channels, seed=w, free_only=False)
    motions = [random_motion(rng, 0.3, 0.3, 0.2) for _ in range(3)] + [(0.1, 0.0, 0.0)]
    ctx.set_fast(fast)
    try:
        _run_pair(ctx, port, occ, channels, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED, B0=B0)
        _run_pair(ctx, port, occ, channels, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED)
    finally:
        ctx.set_fast(True)


@pytest.mark.parametrize("fast", [True, False])
def test_fast_and_strict_variants_agree(ctx, port, fast):
    """The FAST fused variant (clean tensors) and the literal STRICT sequence
    are both bit-exact against the oracle."""
    occ = make_floorplan(130, 70, seed=12)
    rng = Rng(3)
    motions = [random_motion(rng) for _ in range(4)] + [(0.1, 0.0, 0.0), (0.2, 0.1, 0.0)]
    ctx.set_fast(fast)
    try:
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED)
        _run_pair(ctx, port, occ, 72, (1e-4, 1e-4, 0.012), motions, GL_PATH_FUSED)
    finally:
        ctx.set_fast(True)


def test_unclean_inputs_bit_exact(ctx, port):
    """Uploaded tensors with -0.0 and negative values are detected and run
    the strict variant: still bit-identical, including integral shifts."""
    occ = make_floorplan(96, 64, seed=13)
    B0 = random_tensor(occ, 72, seed=5, free_only=False) - 0.3
    B0[0, 10:20, 10:20] = -0.0
    motions = [(0.1, 0.0, 0.0), (0.2, 0.1, 0.0), (0.05, 0.03, 0.02)]
    for path in (GL_PATH_FUSED, GL_PATH_GENERIC):
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, path, B0=B0)


def test_large_shifts_bit_exact(ctx, port):
    """Multi-cell and far-out-of-grid shifts (observe() can flush any motion)."""
    occ = make_floorplan(96, 64, seed=9)
    motions = [(0.95, -0.4, 0.0), (3.3, 2.1, 0.2), (-40.0, 0.0, 0.0), (0.1, 0.0, 0.0)]
    B0 = random_tensor(occ, 72, seed=2)
    for path in (GL_PATH_FUSED, GL_PATH_GENERIC):
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, path, B0=B0)


def test_rescale_branch_bit_exact(ctx, port):
    """max < 1e-6 -> uniform rescale (belief_tensor.cpp:486-493), applied
    lazily by the next reader; results must stay identical."""
    occ = make_floorplan(96, 80, seed=2)
    B0 = random_tensor(occ, 72, seed=3) * 1e-9
    motions = [(0.05, 0.01, 0.02), (0.1, 0.0, 0.0), (0.0, 0.0, 0.1)]
    for path in (GL_PATH_FUSED, GL_PATH_GENERIC):
        t, B = _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, path, B0=B0)
        assert B.max() == 1.0 or B.max() > 1e-6


def test_extinguish_raises(ctx, port):
    """test_belief_engine.cpp:321-335: all mass pushed into a wall."""
    occ = np.ones((8, 8), np.uint8)
    occ[3, 3] = 0
    for path in (GL_PATH_FUSED, GL_PATH_GENERIC):
        _run_pair(ctx, port, occ, 4, (0.001, 0.001, 0.0001), [(0.4, 0.0, 0.0)], path)


def test_bare_impulse_into_wall_extinguishes(ctx, port):
    """test_belief_engine.cpp:307-319."""
    occ = make_empty_room(24, 24)
    B0 = np.zeros((8, 24, 24))
    B0[0, 12, 22] = 1.0
    for path in (GL_PATH_AUTO, GL_PATH_GENERIC):
        _run_pair(ctx, port, occ, 8, (0.05, 0.05, 0.05), [(0.1, 0.0, 0.0)], path, B0=B0)


def test_trace_256x256x36_200_steps(ctx, port, ref):
    """Config 1: 256^2 x 36 floor plan, 200 steps of a recorded Localizer
    trace (both kernel slots), bit-exact after every step via device hash."""
    import oracle
    occ = make_floorplan(256, 256, seed=0)
    rm = oracle.RefMap(ref, occ=occ)
    js, is_ = np.nonzero(occ == 0)
    start = (is_[len(is_) // 2] * 0.1 + 0.05, js[len(js) // 2] * 0.1 + 0.05, 0.3)
    ev, _ = oracle.ref_gen_trace(ref, rm, 36, start, seed=3, max_steps=200)
    steps = ev[ev[:, 0] == 0]
    assert len(steps) == 200
    m, ks, act = _setup(ctx, occ, 36, (0.03, 0.03, 0.012))
    _, rks, ract = _setup(ctx, occ, 36, (1e-4, 1e-4, 0.012))
    cells = m.cells()
    pk = [port.build_kernels(0.03, 0.03, 0.012, 36, 0.1), port.build_kernels(1e-4, 1e-4, 0.012, 36, 0.1)]
    pinv = [port.make_activation(cells, k, 36)[1] for k in pk]
    t = g.init_uniform(m, 36, ctx)
    B = port.init_uniform(cells, 36)
    th = 0.0
    for s, e in enumerate(steps):
        slot = int(e[4])
        rc, th = port.step(B, th, e[1], e[2], e[3], cells, 0.1, pk[slot], pinv[slot])
        assert rc == 0
        g.step(t, g.OdometryDelta(e[1], e[2], e[3]), m, (ks, rks)[slot], (act, ract)[slot], ctx)
        assert t.hash() == g.tensor_hash_host(B), f"hash mismatch at step {s}"
    assert t.theta_t() == th
    assert_bitwise(t.values(), B, "final")


def test_channel_windows_bit_exact(ctx, port):
    """Theta = 400 (h = 3): the fused launch carries at most kParamChannels
    shift records, so the step runs as two channel-window launches; the max
    (and the rescale branch) is finalised once, by the last window. Small
    grids also split every tile's channels into chunks (each recomputing its
    2H angular neighbours) — every case here runs chunked."""
    occ = make_floorplan(64, 48, seed=21)
    motions = [(0.1, 0.0, 0.0), (0.07, -0.03, 0.05), (0.0, 0.0, 0.02)]
    _run_pair(ctx, port, occ, 400, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED)
    B0 = random_tensor(occ, 400, seed=4) * 1e-9  # max < 1e-6: deferred rescale
    _run_pair(ctx, port, occ, 400, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED, B0=B0)


@pytest.mark.parametrize("chunks", [1, 2, 3, 7])
@pytest.mark.parametrize("channels", [72, 360])
def test_explicit_channel_chunks_bit_exact(ctx, port, chunks, channels):
    """gl_context_set_channel_chunks: any split of the channel walk (each
    chunk recomputing its 2H angular neighbours) gives the same bits."""
    occ = make_floorplan(96, 64, seed=8)
    rng = Rng(chunks * 7 + channels)
    motions = [random_motion(rng) for _ in range(3)]
    ctx.set_channel_chunks(chunks)
    try:
        _run_pair(ctx, port, occ, channels, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED)
    finally:
        ctx.set_channel_chunks(0)


@pytest.mark.parametrize("tail", [(1, 2), (5, 3), (100000, 2), (0, 2)])
@pytest.mark.parametrize("channels", [72, 360])
def test_wave_tail_split_bit_exact(ctx, port, tail, channels):
    """gl_context_set_wave_tail: the grid's last CTAs splitting their tiles'
    channels (up to every CTA) gives the same bits as the unsplit walk."""
    occ = make_floorplan(200, 120, seed=5)
    rng = Rng(tail[0] + channels)
    motions = [random_motion(rng) for _ in range(3)]
    ctx.set_channel_chunks(1)
    ctx.set_wave_tail(*tail)
    try:
        _run_pair(ctx, port, occ, channels, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED)
    finally:
        ctx.set_wave_tail(-1, 3)
        ctx.set_channel_chunks(0)


@pytest.mark.parametrize("himax", [1, 2])
def test_high_word_max_modes_bit_exact(ctx, port, himax):
    """The fused FAST kernel's high-word max (forced on small tensors here;
    automatic on >= 2^27 states) must give the reference's status and
    pending rescale: decisive steps, the rescale branch (max < 1e-6, taken by
    the exact full-grid epilogue) and extinguish, every step bit-exact."""
    occ = make_floorplan(96, 80, seed=2)
    ctx.set_himax(himax)
    try:
        rng = Rng(9)
        motions = [random_motion(rng) for _ in range(3)] + [(0.1, 0.0, 0.0), (0.0, 0.0, 0.1)]
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED)
        B0 = random_tensor(occ, 72, seed=3) * 1e-9  # rescale every step
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions, GL_PATH_FUSED, B0=B0)
        B0 = random_tensor(occ, 72, seed=4) * 1e-300  # denormal range: hi words near 0
        _run_pair(ctx, port, occ, 72, (0.03, 0.03, 0.012), motions[:2], GL_PATH_FUSED, B0=B0)
        occx = np.ones((8, 8), np.uint8)
        occx[3, 3] = 0
        _run_pair(ctx, port, occx, 4, (0.001, 0.001, 0.0001), [(0.4, 0.0, 0.0)], GL_PATH_FUSED)
    finally:
        ctx.set_himax(0)


def _custom_kernels(ctx, port, channels, sep, ang):
    """The same explicit KernelSet for the GPU and the oracle."""
    import oracle
    sep = np.asarray(sep, np.float64)
    dense = np.outer(sep, sep).ravel()
    spatial = np.tile(dense, channels)
    ks = g.KernelSet.from_arrays(1, True, sep, spatial, ang, channels, ctx=ctx)
    pks = oracle.Kernels(1, True, sep, spatial, [a[0] for a in ang], [a[1] for a in ang])
    return ks, pks


@pytest.mark.parametrize("symmetric", [True, False])
def test_custom_tap_sets_route_by_symmetry(ctx, port, symmetric):
    """v10's product sharing needs bitwise-symmetric taps (fused_supported
    checks it); an asymmetric user KernelSet must fall back to the generic
    chain and stay bit-exact, and forcing the fused path must fail loudly."""
    occ = make_floorplan(96, 80, seed=21)
    C_ = 24
    if symmetric:
        sep, ang = [0.25, 0.5, 0.25], [(-1, 0.2), (0, 0.6), (1, 0.2)]
    else:
        sep, ang = [0.2, 0.5, 0.3], [(-1, 0.1), (0, 0.6), (1, 0.3)]
    ks, pks = _custom_kernels(ctx, port, C_, sep, ang)
    h, w = occ.shape
    m = g.OccupancyMap(w, h, 0.1, occ, ctx=ctx)
    act = g.make_activation(m, ks, C_, ctx)
    cells = m.cells()
    _, pinv = port.make_activation(cells, pks, C_)
    rng = Rng(5)
    motions = [random_motion(rng) for _ in range(4)]
    for path in (GL_PATH_AUTO, GL_PATH_FUSED):
        ctx.set_path(path)
        try:
            t = g.init_uniform(m, C_, ctx)
            B = port.init_uniform(cells, C_)
            th = 0.0
            for (u, v, w_) in motions:
                rc, th = port.step(B, th, u, v, w_, cells, 0.1, pks, pinv)
                assert rc == 0
                if path == GL_PATH_FUSED and not symmetric:
                    with pytest.raises(ValueError):
                        g.step(t, g.OdometryDelta(u, v, w_), m, ks, act, ctx)
                    break
                g.step(t, g.OdometryDelta(u, v, w_), m, ks, act, ctx)
            else:
                assert_bitwise(t.values(), B, f"custom taps symmetric={symmetric} path={path}")
        finally:
            ctx.set_path(GL_PATH_AUTO)
