#!/usr/bin/env python
"""One configs[2] observation cycle after a warm-up of N steps with the
cmd_bench cadence (experiment only; run under `ncu` for the cycle's launch
list: the cycle is bracketed by cudaProfilerStart/Stop)."""
import ctypes
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1910_00572_b200 as g  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
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
    for s in range(n):
        g.step_async(t, u, m, ks, act, ctx)
        if s % every == 0:
            g.observation_update(t, g.dither_samples(t, 512), scan, m, f, lp)
    g.step_async(t, u, m, ks, act, ctx)
    ctx.synchronize()
    cudart = ctypes.CDLL("libcudart.so") if False else None
    import torch
    torch.cuda.cudart().cudaProfilerStart()
    smp = g.dither_samples(t, 512)
    g.observation_update(t, smp, scan, m, f, lp)
    g.step_async(t, u, m, ks, act, ctx)
    ctx.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("samples", len(smp.cells))


if __name__ == "__main__":
    main()
