#!/usr/bin/env python
"""Time the pieces of one LIDAR observation cycle at 1024^2x72 on the GPU
(belief_map, dither on a host plane, dither from the tensor, observation
update) with host wall clocks around synchronous calls."""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, simple_scan, write_pgm  # noqa: E402


def t(fn, n=3):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), r


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    C = 72
    ctx = g.Context(0)
    occ = make_floorplan(W, W, seed=0)
    m = g.load_map(write_pgm(occ), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    tt = g.init_uniform(m, C, ctx)
    for _ in range(5):
        g.step(tt, g.OdometryDelta(0.1, 0.0, 0.02), m, ks, act, ctx)
    f = g.DistanceField(m, ctx)
    js, is_ = np.nonzero(occ == 0)
    a, r = simple_scan(occ, is_[len(is_) // 2] * 0.1 + 0.05, js[len(js) // 2] * 0.1 + 0.05, 0.3)
    scan = g.LidarScan(a, r, 8.0)
    ms_bm, bm = t(lambda: g.belief_map(tt))
    ms_dh, s = t(lambda: g.dither_samples(bm, 512, ctx))
    ms_dt, s2 = t(lambda: g.dither_samples(tt, 512))
    ms_ob, _ = t(lambda: g.observation_update(tt, s2, scan, m, f, g.LikelihoodParams()), n=2)
    print(f"W={W}: belief_map {ms_bm:.2f} ms | dither(host plane) {ms_dh:.2f} ms | "
          f"dither(tensor) {ms_dt:.2f} ms | observation_update {ms_ob:.2f} ms | samples {len(s2.cells)}")


if __name__ == "__main__":
    main()
