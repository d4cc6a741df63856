#!/usr/bin/env python
"""Host cost of one step call at configs[0] (256^2 x 36; experiment only):
enqueue-only time of step_async (before the stream sync), the synchronous
g.step, and the raw C-ABI call through ctypes without the Python wrapper."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 36
    ctx = g.Context(0)
    m = g.load_map(write_pgm(make_floorplan(W, W, seed=0)), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(0.1, 0.0, 0.0)
    for _ in range(50):
        g.step(t, u, m, ks, act, ctx)
    n = 300
    lib = ctx.lib
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(n):
            g.step_async(t, u, m, ks, act, ctx)
        t1 = time.perf_counter()
        ctx.synchronize()
        t2 = time.perf_counter()
        for _ in range(n):
            lib.gl_step_async(ctx.h, t.h, u.u, u.v, u.w, m.h, ks.h, act.h)
        t3 = time.perf_counter()
        ctx.synchronize()
        t4 = time.perf_counter()
        for _ in range(n):
            g.step(t, u, m, ks, act, ctx)
        t5 = time.perf_counter()
        print(f"W={W} C={C}: step_async enqueue {1e6*(t1-t0)/n:.2f} us | raw C-ABI enqueue {1e6*(t3-t2)/n:.2f} us | "
              f"sync step {1e6*(t5-t4)/n:.2f} us | device-bound async {1e6*(t2-t0)/n:.2f} us")


if __name__ == "__main__":
    main()
