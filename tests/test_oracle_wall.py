"""CPU checks of the wall-crossing rule's restatement (oracle/gl_oracle.c
glo_seg_cells / glo_step_wall; the rule is an extension, see
tests/test_gpu_wall_mask.py): hand-derived known answers, a dense-sampling
cross-check of the exact integer crossing test, and the rule's invariants."""
import math

import numpy as np
import pytest

from tests.helpers import make_floorplan


KNOWN = {
    (1, 0): [], (1, 1): [], (2, 0): [(-1, 0)], (2, 2): [(-1, -1)],
    (2, 1): [(-1, -1), (-1, 0)], (-2, 1): [(1, -1), (1, 0)], (0, -3): [(0, 1), (0, 2)],
    (3, 2): [(-2, -2), (-2, -1), (-1, -1), (-1, 0)],
}


@pytest.mark.parametrize("o", sorted(KNOWN))
def test_seg_cells_known_answers(port, o):
    cells, n = port.seg_cells(*o)
    assert n == len(KNOWN[o]) and sorted(cells) == sorted(KNOWN[o])


def _sampled(ox, oy, samples=20000):
    """Cells whose open interior a dense sampling of the open segment hits
    (interior = distance to the cell centre < 1/2 - eps on both axes)."""
    out = set()
    eps = 1e-9
    for s in range(1, samples):
        t = s / samples
        x, y = t * ox, t * oy
        cx, cy = math.floor(x + 0.5), math.floor(y + 0.5)
        if abs(x - cx) < 0.5 - eps and abs(y - cy) < 0.5 - eps:
            out.add((cx - ox, cy - oy))
    out.discard((0, 0))
    out.discard((-ox, -oy))
    return out


@pytest.mark.parametrize("ox,oy", [(ox, oy) for ox in range(-4, 5) for oy in range(-4, 5)])
def test_seg_cells_match_dense_sampling(port, ox, oy):
    cells, n = port.seg_cells(ox, oy)
    assert set(cells) == _sampled(ox, oy)


def test_wall_step_equals_plain_step_on_an_open_map(port):
    """Without interior walls no tap is blocked away from the boundary ring:
    the masked step equals the reference step wherever the ring cannot be
    crossed (every tap of a free cell inside the ring stays inside it)."""
    occ = np.zeros((40, 48), np.uint8)
    occ[0, :] = occ[-1, :] = 1
    occ[:, 0] = occ[:, -1] = 1
    ks = port.build_kernels(0.03, 0.03, 0.012, 16, 0.1)
    _, inv = port.make_activation(occ, ks, 16)
    A = port.init_uniform(occ, 16)
    B = A.copy()
    port.step(A, 0.0, 0.13, 0.07, 0.1, occ, 0.1, ks, inv)
    port.step(B, 0.0, 0.13, 0.07, 0.1, occ, 0.1, ks, inv, wall=True)
    assert np.array_equal(A.view(np.uint64), B.view(np.uint64))


def test_wall_step_never_adds_mass(port):
    """Dropping taps only removes terms: the masked step is <= the plain
    one cell by cell (same positive activation inverse)."""
    occ = make_floorplan(64, 48, seed=6)
    ks = port.build_kernels(0.03, 0.03, 0.012, 16, 0.1)
    _, inv = port.make_activation(occ, ks, 16)
    A = port.init_uniform(occ, 16)
    B = A.copy()
    port.step(A, 0.0, 0.3, -0.2, 0.1, occ, 0.1, ks, inv)
    port.step(B, 0.0, 0.3, -0.2, 0.1, occ, 0.1, ks, inv, wall=True)
    assert (B <= A).all() and (B < A).any()
