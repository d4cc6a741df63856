#!/usr/bin/env python
"""Wall time of the read-outs on a configs[2]-state belief (experiment only):
argmax_state (exact confidence total over the tensor), belief_map,
tensor hash, after N steps with the cmd_bench observation cadence."""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1910_00572_b200 as g  # noqa: E402


def t(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


def main():
    W = H = 1024
    C, every = 72, 16
    ctx = g.Context(0)
    m = g.load_map(bench.make_map_bytes(W, H), 250, 0.1, ctx=ctx)
    f = g.DistanceField(m, ctx)
    ks = g.build_kernels(g.MotionNoise(), C, m.resolution(), 2.0 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    tt = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)
    a, r = bench.lidar_scan(W, H)
    scan = g.LidarScan(a, r, 8.0)
    lp = g.LikelihoodParams()
    for n in (0, 32, 160):
        for s in range(n):
            g.step_async(tt, u, m, ks, act, ctx)
            if s % every == 0:
                g.observation_update(tt, g.dither_samples(tt, 512), scan, m, f, lp)
        ctx.synchronize()
        print(f"after {n} more steps: argmax_state {t(lambda: g.argmax_state(tt)):.3f} ms | "
              f"step {t(lambda: g.step(tt, u, m, ks, act, ctx)):.3f} ms")


if __name__ == "__main__":
    main()
