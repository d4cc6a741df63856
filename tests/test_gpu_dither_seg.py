"""The segment-parallel Floyd-Steinberg sweep (k_dither_seg: row segments run
by the lanes of one warp from a guessed carry, verified bitwise against the
previous segment's true error and rerun until the chains meet) against the
oracle's sequential dither_samples (observation.cpp:11-71): sample lists in
emission order and source masses bit-identical on planes chosen to stress
every path — sparse and dense emissions (many per segment), segments that
need a rerun, reruns that run through their segment (isolated spikes whose
error tails cross exact-zero runs, steep exponential tails: several
verification rounds), widths from the narrowest that segments to the
shared-memory limit, long thin and tall planes."""
import numpy as np
import pytest

import paper_1910_00572_b200 as g

pytestmark = pytest.mark.gpu


def _plane(kind, w, h, seed):
    rng = np.random.default_rng(seed)
    if kind == "sparse":       # a converged belief: few emissions per row
        bm = rng.random((h, w)) ** 12
    elif kind == "dense":      # many emissions per row and segment
        bm = rng.random((h, w))
    elif kind == "blobs":      # localized mass, most of the plane zero
        bm = np.zeros((h, w))
        for _ in range(6):
            cy, cx = rng.integers(0, h), rng.integers(0, w)
            yy, xx = np.mgrid[0:h, 0:w]
            bm += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2.0 * rng.uniform(2, 30) ** 2))
    elif kind == "walls":      # a floor plan's support: zero rows / columns
        bm = rng.random((h, w)) ** 4
        bm[:, ::37] = 0.0
        bm[::23, :] = 0.0
    elif kind == "spikes":     # isolated masses in exact zeros: long decaying error tails
        bm = np.zeros((h, w))
        n = max(1, w // 300)
        for j in range(h):
            bm[j, rng.integers(0, w, n)] = rng.uniform(0.5, 3.0, n)
    elif kind == "tails":      # steep exponential profiles over many decades
        xx = np.arange(w)[None, :]
        cx = rng.integers(0, w, (h, 1))
        bm = np.exp(-np.abs(xx - cx) * rng.uniform(0.5, 3.0, (h, 1))) * rng.uniform(0.1, 1.0, (h, 1))
    else:
        raise KeyError(kind)
    return bm


@pytest.mark.parametrize("kind", ["sparse", "dense", "blobs", "walls", "spikes", "tails"])
@pytest.mark.parametrize("w,h,budget", [(128, 40, 64), (200, 64, 512), (1000, 30, 512), (1024, 64, 4096),
                                        (2048, 16, 512), (4096, 6, 20000), (333, 333, 100000)])
def test_segment_sweep_bit_exact(ctx, port, kind, w, h, budget):
    bm = _plane(kind, w, h, w * 31 + h)
    s = g.dither_samples(bm, budget, ctx)
    cells, mass = port.dither(bm, budget)
    assert s.source_mass == mass
    assert np.array_equal(s.cells, cells), (len(s.cells), len(cells))


def test_segment_sweep_on_a_floorplan_belief(ctx, port):
    """A 1024^2 belief map after a few steps (the LIDAR cycle's input)."""
    import math
    from paper_1910_00572_b200.floorplan import make_floorplan
    occ = make_floorplan(1024, 1024, seed=0)
    m = g.OccupancyMap(1024, 1024, 0.1, occ, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), 72, 0.1, 2 * math.pi / 72)
    act = g.make_activation(m, ks, 72, ctx)
    t = g.init_uniform(m, 72, ctx)
    for (u, v, w_) in [(0.1, 0.0, 0.0), (0.05, 0.02, 0.1)] * 3:
        g.step(t, g.OdometryDelta(u, v, w_), m, ks, act, ctx)
    bm = g.belief_map(t)
    for budget in (512, 20000):
        s = g.dither_samples(t, budget)
        cells, mass = port.dither(bm, budget)
        assert s.source_mass == mass
        assert np.array_equal(s.cells, cells)


def test_segment_sweep_randomised(ctx, port):
    """300 random (width, height, plane kind, budget) draws incl. exact-zero
    rows and widths past the shared-memory limit of the segment sweep (its
    fallbacks); tools/stress_dither.py runs the same draw at 3000 cases."""
    rng = np.random.default_rng(12345)
    kinds = ["sparse", "dense", "blobs", "walls", "spikes", "tails"]
    for i in range(300):
        w = int(rng.integers(200, 7000)) if rng.random() < 0.3 else int(rng.integers(200, 1500))
        h = int(rng.integers(1, 60))
        budget = int(rng.choice([16, 512, 4096, 100000]))
        bm = _plane(kinds[i % len(kinds)], w, h, int(rng.integers(1 << 30)))
        if rng.random() < 0.2:
            bm[rng.integers(0, h, 3), :] = 0.0
        s = g.dither_samples(bm, budget, ctx)
        cells, mass = port.dither(bm, budget)
        assert s.source_mass == mass, (i, w, h, budget)
        assert np.array_equal(s.cells, cells), (i, w, h, budget, len(s.cells), len(cells))
