"""dither_samples' total (observation.cpp:16-17: total = 0.0; total += v in
row-major order) computed by the device's parallel binade scan
(k_observe.cu k_seq_sum) must equal the sequential FP64 chain bit for bit:
ties to even at every ulp scale, binade crossings mid-chunk and at chunk
edges, subnormals, huge dynamic range, zeros and -0.0, and the 1024^2
LIDAR-cycle plane sizes. Out-of-domain inputs (negative, inf, NaN) are
rejected (the dither kernel then runs its sequential chain)."""
import numpy as np
import pytest

import paper_1910_00572_b200 as g

pytestmark = pytest.mark.gpu


def seq(x):
    t = 0.0
    for v in np.asarray(x, dtype=np.float64).tolist():
        t += v
    return t


def _eq(a, b):
    return np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


CASES = {
    "random_uniform_1e5": lambda r: r.random(100_000),
    "random_pow8_with_zeros": lambda r: np.where(r.random(300_000) < 0.3, 0.0, r.random(300_000) ** 8),
    "ties_half_ulp": lambda r: np.concatenate([[1.0], np.full(20000, 2.0 ** -53), r.integers(1, 7, 20000) * 2.0 ** -53]),
    "ties_many_scales": lambda r: np.concatenate([[1.5], (r.integers(0, 8, 50000) * 0.5 + 0.5) * 2.0 ** -52,
                                                 (r.integers(0, 8, 50000) * 0.5 + 0.5) * 2.0 ** -50]),
    "subnormals_then_normals": lambda r: np.concatenate([r.integers(0, 5, 30000) * 5e-324, r.random(30000) * 1e-300,
                                                        r.random(10000)]),
    "dynamic_range": lambda r: 10.0 ** r.uniform(-30, 30, 200_000),
    "growing_crossing_every_chunk": lambda r: 2.0 ** np.arange(0, 60, 0.0004)[:150_000],
    "single_and_empty_prefix": lambda r: np.concatenate([np.zeros(70_000), [3.0], np.zeros(10), [0.25]]),
    "minus_zero": lambda r: np.concatenate([[-0.0, 0.0, -0.0], r.random(5000), [-0.0] * 7, r.random(9000)]),
    "all_zero": lambda r: np.zeros(12345),
    "long_zero_prefix": lambda r: np.concatenate([np.where(r.random(9_000_000) < 1e-6, -0.0, 0.0), [2.0 ** -1070],
                                                  np.zeros(100_000), r.random(50_000) ** 20]),
    "many_crossings_per_chunk": lambda r: 2.0 ** np.linspace(-1070, 10, 400_000) * r.random(400_000),
    "crossings_and_ties": lambda r: np.concatenate([2.0 ** np.linspace(-60, 0, 30_000) * r.random(30_000),
                                                    r.integers(0, 4, 30_000) * 2.0 ** -54]),
    # a binade crossing in every one of ~600 chunks: more crossing chunks
    # than the all-SM event pass has slots (512), so the walk's own pass
    # takes the rest
    "crossing_chunks_beyond_pool": lambda r: 2.0 ** (-1000.0 + np.arange(600 * 8192) / 8192.0)
    * (0.5 + 0.5 * r.random(600 * 8192)),
    "plane_1024sq": lambda r: np.where(r.random(1 << 20) < 0.16, 0.0, r.random(1 << 20) ** 3),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_sequential_sum_bit_exact(ctx, name):
    x = np.ascontiguousarray(CASES[name](np.random.default_rng(len(name))), dtype=np.float64)
    got = g.sequential_sum(x, ctx)
    want = seq(x)
    assert _eq(got, want), (name, got, want)


@pytest.mark.parametrize("bad", [-1.0, np.inf, np.nan])
def test_out_of_domain_rejected(ctx, bad):
    x = np.ones(1000)
    x[500] = bad
    with pytest.raises(ValueError):
        g.sequential_sum(x, ctx)


def test_dither_total_on_negative_plane_still_exact(ctx, port):
    """A plane with negative values takes the dither kernel's sequential
    chain for the total: sample list and source mass still bit-exact."""
    rng = np.random.default_rng(5)
    bm = rng.random((64, 80)) - 0.1
    s = g.dither_samples(bm, 128, ctx)
    cells, mass = port.dither(bm, 128)
    assert _eq(s.source_mass, mass) and np.array_equal(s.cells, cells)
