"""Seeded synthetic floor plans and the reference's deterministic RNG.

The reference ships only five small fixed worlds (worlds.cpp, <= 94x56
cells); BASELINE.json's 256^2 / 1024^2 / 4096^2 floor plans are generated
here: rooms-and-corridors by recursive partitioning with 2-cell walls, door
gaps and furniture blocks, 0.1 m/cell, the boundary ring occupied. Maps are
emitted as canonical P5 PGM (free = 255, occupied = 0; the reference's
write_pgm, occupancy_map.cpp:177-185) so that both the GPU path and the CPU
oracle load byte-identical maps through load_map(bytes, 250, 0.1).
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


class Rng:
    """xoshiro256++ with the reference's hand-rolled distributions
    (/root/reference/proj/include/gridloc/rng.hpp:10-74): same seed ->
    same draws, so ported reference tests see identical inputs."""

    def __init__(self, seed: int = 0x9E3779B97F4A7C15):
        self.reseed(seed)

    def reseed(self, seed: int):
        x = seed & _M64
        s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & _M64
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
            s.append(z ^ (z >> 31))
        self.s = s
        self.have_spare = False
        self.spare = 0.0

    @staticmethod
    def _rotl(x, k):
        return ((x << k) | (x >> (64 - k))) & _M64

    def next_u64(self) -> int:
        s = self.s
        result = (self._rotl((s[0] + s[3]) & _M64, 23) + s[0]) & _M64
        t = (s[1] << 17) & _M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = (self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_int(self, n: int) -> int:
        return self.next_u64() % n

    def normal(self, mean: float = 0.0, stddev: float = 1.0) -> float:
        import math
        if self.have_spare:
            self.have_spare = False
            return mean + stddev * self.spare
        while True:
            u = 2.0 * self.uniform() - 1.0
            v = 2.0 * self.uniform() - 1.0
            q = u * u + v * v
            if not (q >= 1.0 or q == 0.0):
                break
        f = math.sqrt(-2.0 * math.log(q) / q)
        self.spare = v * f
        self.have_spare = True
        return mean + stddev * (u * f)


def force_ring(occ: np.ndarray) -> np.ndarray:
    occ[0, :] = 1
    occ[-1, :] = 1
    occ[:, 0] = 1
    occ[:, -1] = 1
    return occ


def make_empty_room(width: int, height: int) -> np.ndarray:
    """worlds.cpp:88-92: free interior, occupied boundary."""
    occ = np.ones((height, width), np.uint8)
    if width > 2 and height > 2:
        occ[1:height - 1, 1:width - 1] = 0
    return occ


def make_floorplan(width: int, height: int, seed: int = 0, room_min: int = 36, room_max: int = 120,
                   wall: int = 2, door: tuple = (8, 14), clutter: float = 0.12) -> np.ndarray:
    """Rooms-and-corridors floor plan, uint8 (H, W), 1 = occupied."""
    rng = Rng(0xF100 + seed)
    occ = np.zeros((height, width), np.uint8)
    force_ring(occ)
    rooms = []
    stack = [(1, 1, width - 2, height - 2)]  # inclusive free region
    while stack:
        x0, y0, x1, y1 = stack.pop()
        rw, rh = x1 - x0 + 1, y1 - y0 + 1
        split_x = rw >= rh
        span = rw if split_x else rh
        if span <= room_max or span < 2 * room_min + wall:
            rooms.append((x0, y0, x1, y1))
            continue
        cut = room_min + int(rng.uniform_int(span - 2 * room_min - wall + 1))
        if split_x:
            wx = x0 + cut
            occ[y0:y1 + 1, wx:wx + wall] = 1
            _doors(occ, rng, (y0, y1), lambda a, b: occ.__setitem__((slice(a, b), slice(wx, wx + wall)), 0), door)
            stack.append((x0, y0, wx - 1, y1))
            stack.append((wx + wall, y0, x1, y1))
        else:
            wy = y0 + cut
            occ[wy:wy + wall, x0:x1 + 1] = 1
            _doors(occ, rng, (x0, x1), lambda a, b: occ.__setitem__((slice(wy, wy + wall), slice(a, b)), 0), door)
            stack.append((x0, y0, x1, wy - 1))
            stack.append((x0, wy + wall, x1, y1))
    # furniture: axis-aligned blocks away from walls
    for (x0, y0, x1, y1) in rooms:
        area = (x1 - x0 + 1) * (y1 - y0 + 1)
        target = clutter * area
        placed = 0
        tries = 0
        while placed < target and tries < 40:
            tries += 1
            bw = 3 + int(rng.uniform_int(10))
            bh = 3 + int(rng.uniform_int(10))
            if x1 - x0 - bw - 6 <= 0 or y1 - y0 - bh - 6 <= 0:
                break
            bx = x0 + 3 + int(rng.uniform_int(x1 - x0 - bw - 5))
            by = y0 + 3 + int(rng.uniform_int(y1 - y0 - bh - 5))
            occ[by:by + bh, bx:bx + bw] = 1
            placed += bw * bh
    return force_ring(occ)


def _doors(occ, rng, span, carve, door):
    lo, hi = span
    n = 1 + int(rng.uniform_int(2))
    for _ in range(n):
        dw = door[0] + int(rng.uniform_int(door[1] - door[0] + 1))
        if hi - lo + 1 <= dw + 2:
            carve(lo, hi + 1)
            return
        a = lo + 1 + int(rng.uniform_int(hi - lo - dw))
        carve(a, a + dw)


def simple_scan(occ: np.ndarray, x: float, y: float, theta: float, beams: int = 24, max_range: float = 8.0,
                res: float = 0.1):
    """A noise-free full-circle scan by fixed-step ray marching (synthetic
    bench input; the reference's exact grid traversal lives in its
    simulator, occupancy_map.cpp:273-332)."""
    import math
    angles = np.array([-math.pi + b * (2.0 * math.pi / beams) for b in range(beams)])
    ranges = np.full(beams, max_range)
    h, w = occ.shape
    for b, a in enumerate(angles):
        c, s = math.cos(theta + a), math.sin(theta + a)
        r = 0.0
        while r < max_range:
            i, j = int(math.floor((x + r * c) / res)), int(math.floor((y + r * s) / res))
            if not (0 <= i < w and 0 <= j < h) or occ[j, i]:
                ranges[b] = r
                break
            r += 0.25 * res
    return angles, ranges


def write_pgm(occ: np.ndarray) -> bytes:
    """Canonical P5 (occupancy_map.cpp:177-185): free 255, occupied 0."""
    h, w = occ.shape
    header = f"P5\n{w} {h}\n255\n".encode()
    return header + np.where(occ != 0, 0, 255).astype(np.uint8).tobytes()


def free_cells(occ: np.ndarray):
    js, is_ = np.nonzero(occ == 0)
    return is_, js
