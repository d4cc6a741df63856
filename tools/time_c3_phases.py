#!/usr/bin/env python
"""Phase wall times of the configs[2] loop (experiment only): synchronous
steps, dither_samples(tensor), observation_update, in the sync and the async
loop, to locate where the end-to-end loop spends its time."""
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
    pgm = bench.make_map_bytes(W, H)
    m = g.load_map(pgm, 250, 0.1, ctx=ctx)
    f = g.DistanceField(m, ctx)
    ks = g.build_kernels(g.MotionNoise(), C, m.resolution(), 2.0 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)
    a, r = bench.lidar_scan(W, H)
    scan = g.LidarScan(a, r, 8.0)
    lp = g.LikelihoodParams()
    for sync in (False, True, False, True):
        ph = {"step": [], "step_after_obs": [], "dither": [], "obs": []}
        after = False
        t00 = time.perf_counter()
        for s in range(160):
            t0 = time.perf_counter()
            (g.step if sync else g.step_async)(t, u, m, ks, act, ctx)
            ph["step_after_obs" if after else "step"].append(time.perf_counter() - t0)
            after = False
            if s % every == 0:
                t0 = time.perf_counter()
                smp = g.dither_samples(t, 512)
                t1 = time.perf_counter()
                g.observation_update(t, smp, scan, m, f, lp)
                t2 = time.perf_counter()
                ph["dither"].append(t1 - t0)
                ph["obs"].append(t2 - t1)
                after = True
        ctx.synchronize()
        tot = time.perf_counter() - t00
        print(f"sync={sync}: {160 / tot:.0f} Hz; " + "; ".join(
            f"{k} med {1e3 * np.median(v):.3f} ms sum {1e3 * np.sum(v):.1f} ms" for k, v in ph.items()))


if __name__ == "__main__":
    main()
