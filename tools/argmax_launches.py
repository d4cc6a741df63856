#!/usr/bin/env python
"""argmax_state on a configs[2]-state belief under cudaProfilerStart/Stop
(experiment only: run under ncu for its launch list)."""
import math
import os
import sys

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
    tt = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(m.resolution(), 0.0, 0.0)
    a, r = bench.lidar_scan(W, H)
    scan = g.LidarScan(a, r, 8.0)
    for s in range(64):
        g.step_async(tt, u, m, ks, act, ctx)
        if s % every == 0:
            g.observation_update(tt, g.dither_samples(tt, 512), scan, m, f, g.LikelihoodParams())
    g.argmax_state(tt)
    ctx.synchronize()
    import torch
    torch.cuda.cudart().cudaProfilerStart()
    e = g.argmax_state(tt)
    torch.cuda.cudart().cudaProfilerStop()
    print(e)


if __name__ == "__main__":
    main()
