"""Floyd-Steinberg (dither_samples, observation.cpp:11-71) on very wide
maps: rows of >6.3K cells leave the pipelined kernel for the one-warp row
kernel (row buffers in shared memory), and rows of >12.8K cells (2 x W
doubles > 200 KB) put its row buffers in global memory. Bit-exact sample
list and source mass against the oracle on all three paths."""
import numpy as np
import pytest

import paper_1910_00572_b200 as g

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("w,h", [(6000, 6), (9000, 5), (16384, 4), (20000, 3)])
def test_wide_rows_bit_exact(ctx, port, w, h):
    rng = np.random.default_rng(w)
    bm = rng.random((h, w)) ** 4
    bm[rng.random((h, w)) < 0.3] = 0.0
    s = g.dither_samples(bm, 512, ctx)
    cells, mass = port.dither(bm, 512)
    assert s.source_mass == mass
    assert np.array_equal(s.cells, cells), (len(s.cells), len(cells))
    assert len(cells) > 0
