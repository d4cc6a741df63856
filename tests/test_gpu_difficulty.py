"""map_difficulty (evaluation.cpp:25-72) on the device against the
reference's own map_difficulty (compiled from its sources, oracle/_ref):
identical fractions on the reference's fixed worlds and on seeded floor
plans, with its default DifficultyConfig (evaluation.hpp:21-29) and
variations (stride, beam count, partial field of view, theta bins)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle
import paper_1910_00572_b200 as g
from paper_1910_00572_b200._lib import DifficultyC, LikelihoodC, check
from tests.helpers import make_floorplan, random_map

pytestmark = pytest.mark.gpu

DEFAULT = dict(thr=1.0, beams=8, fov=2 * math.pi, max_range=8.0, stride=1, bins=8, lik=(0.2, 0.05, 1))


def _ours(ctx, occ, cfg):
    h, w = occ.shape
    m = g.OccupancyMap(w, h, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    c = DifficultyC(cfg["thr"], cfg["beams"], cfg["fov"], cfg["max_range"], cfg["stride"], cfg["bins"],
                    LikelihoodC(*cfg["lik"]))
    out = C.c_double()
    check(ctx.lib.gl_map_difficulty(ctx.h, m.h, f.h, C.byref(c), C.byref(out)))
    return out.value


def _reference(ref, occ, cfg):
    rm = oracle.RefMap(ref, occ=occ)
    return oracle.ref_map_difficulty(ref, rm, cfg)


def _world(ref, which):
    return oracle.ref_world_cells(ref, which)


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_reference_worlds(ctx, ref, which):
    occ = _world(ref, which)
    assert _ours(ctx, occ, DEFAULT) == _reference(ref, occ, DEFAULT)


@pytest.mark.parametrize("variant", [
    dict(stride=2),
    dict(beams=24, bins=12),
    dict(fov=math.pi, beams=9),
    dict(beams=1),
    dict(bins=1, thr=0.25),
    dict(max_range=1.5),
    dict(lik=(0.1, 0.2, 2)),
])
def test_config_variants(ctx, ref, variant):
    cfg = dict(DEFAULT, **variant)
    for occ in (make_floorplan(48, 40, seed=7), random_map(40, 30, 0.15, 3)):
        assert _ours(ctx, occ, cfg) == _reference(ref, occ, cfg)


def test_floorplan_strided(ctx, ref):
    occ = make_floorplan(160, 120, seed=11)
    cfg = dict(DEFAULT, stride=3)
    assert _ours(ctx, occ, cfg) == _reference(ref, occ, cfg)
