#!/usr/bin/env python
"""dither_samples(tensor) wall time after N configs[2] steps (the cmd_bench
cadence; experiment only): median of 20 calls."""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1910_00572_b200 as g  # noqa: E402


def main():
    W = H = 1024
    C, every = 72, 16
    ctx = g.Context(0)
    m = g.load_map(bench.make_map_bytes(W, H), 250, 0.1, ctx=ctx)
    f = g.DistanceField(m, ctx)
    ks = g.build_kernels(g.MotionNoise(), C, m.resolution(), 2.0 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)
    a, r = bench.lidar_scan(W, H)
    scan = g.LidarScan(a, r, 8.0)
    lp = g.LikelihoodParams()
    done = 0
    lib = os.path.basename(os.path.dirname(os.environ.get("GRIDLOC_B200_LIB", "product/x")))
    for target in [int(v) for v in sys.argv[1:]] or [800]:
        for s in range(done, target):
            g.step_async(t, u, m, ks, act, ctx)
            if s % every == 0:
                g.observation_update(t, g.dither_samples(t, 512), scan, m, f, lp)
        done = target
        ctx.synchronize()
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            g.dither_samples(t, 512)
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{lib}: after {target} steps dither(tensor) median {np.median(ts):.3f} ms")


if __name__ == "__main__":
    main()
