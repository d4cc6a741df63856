"""Where does the synchronous step's time go? Per-call wall time of
(A) g.step (enqueue + status read-back + sync), (B) step_async + stream
sync, (C) back-to-back step_async (device-bound), at 1024^2 x 72."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    C = 72
    ctx = g.Context(0)
    m = g.load_map(write_pgm(make_floorplan(W, W, seed=0)), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(0.1, 0.0, 0.0)
    n = 400
    for _ in range(20):
        g.step(t, u, m, ks, act, ctx)
    for rep in range(2):
        t0 = time.perf_counter()
        for _ in range(n):
            g.step(t, u, m, ks, act, ctx)
        a = (time.perf_counter() - t0) / n * 1e6
        t0 = time.perf_counter()
        for _ in range(n):
            g.step_async(t, u, m, ks, act, ctx)
            ctx.synchronize()
        b = (time.perf_counter() - t0) / n * 1e6
        t0 = time.perf_counter()
        for _ in range(n):
            g.step_async(t, u, m, ks, act, ctx)
        ctx.synchronize()
        c = (time.perf_counter() - t0) / n * 1e6
        t0 = time.perf_counter()
        for _ in range(n):
            g.step_async(t, u, m, ks, act, ctx)
        e = (time.perf_counter() - t0) / n * 1e6
        ctx.synchronize()
        print(f"W={W}: step(sync+status) {a:.1f} us | async+sync {b:.1f} us | async pipelined {c:.1f} us | "
              f"host enqueue only {e:.1f} us")


if __name__ == "__main__":
    main()
