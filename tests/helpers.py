"""Shared test inputs (maps, tensors, motions), mirroring the reference tests'
builders (proj/tests/test_belief_engine.cpp:16-45, worlds.cpp)."""
from __future__ import annotations

import math

import numpy as np

from paper_1910_00572_b200.floorplan import Rng, force_ring, make_empty_room, make_floorplan


def random_map(w, h, occupied_fraction, seed):
    """test_belief_engine.cpp:26-33: Rng draw per cell, ring forced."""
    rng = Rng(seed)
    occ = np.zeros((h, w), np.uint8)
    flat = occ.reshape(-1)
    for q in range(flat.size):
        flat[q] = 1 if rng.uniform() < occupied_fraction else 0
    return force_ring(occ)


def twin_room_map():
    """worlds.cpp make_twin_room_map (94 x 56)."""
    occ = np.ones((56, 94), np.uint8)

    def carve(i0, j0, i1, j1):
        occ[j0:j1 + 1, i0:i1 + 1] = 0
    carve(2, 4, 91, 9)
    carve(28, 1, 33, 3)
    carve(2, 14, 41, 53)
    carve(52, 14, 91, 53)
    carve(10, 10, 13, 13)
    carve(60, 10, 63, 13)
    return force_ring(occ)


def random_motion(rng: Rng, scale_u=0.15, scale_v=0.1, scale_w=0.3):
    return (rng.uniform(-scale_u, scale_u), rng.uniform(-scale_v, scale_v), rng.uniform(-scale_w, scale_w))


def random_tensor(occ, channels, seed, free_only=True):
    rng = np.random.default_rng(seed)
    h, w = occ.shape
    B = rng.random((channels, h, w))
    if free_only:
        B[:, occ != 0] = 0.0
    return B


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    diff = bits(a) != bits(b)
    if diff.any():
        idx = np.argwhere(diff)
        first = tuple(idx[0])
        raise AssertionError(f"{what}: {diff.sum()} of {diff.size} values differ; first at {first}: "
                             f"{a[first]!r} vs {b[first]!r}; max abs {np.abs(a - b).max():.3e}")


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / max(np.abs(b).sum(), 1e-300))


__all__ = ["random_map", "twin_room_map", "random_motion", "random_tensor", "assert_bitwise", "rel_l1",
           "make_empty_room", "make_floorplan", "Rng", "math", "bits"]
