"""Fused step time: TMA box loads (even W) vs the cp.async path (odd W)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200._lib import GL_PATH_GENERIC  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm  # noqa: E402


def run(ctx, W, H, C, path=None):
    m = g.load_map(write_pgm(make_floorplan(W, H, seed=0)), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(0.1, 0.0, 0.0)
    if path is not None:
        ctx.set_path(path)
    for _ in range(10):
        g.step_async(t, u, m, ks, act, ctx)
    ctx.synchronize()
    n = 200
    ctx.mark(0)
    for _ in range(n):
        g.step_async(t, u, m, ks, act, ctx)
    ctx.mark(1)
    ctx.synchronize()
    ctx.set_path(0)
    ms = ctx.marks_ms(0, 1) / n
    gbs = (16 * W * H * C + 9 * W * H) / (ms * 1e-3) / 1e9
    return ms, gbs


def main():
    ctx = g.Context(0)
    for (W, H) in [(1024, 1024), (1023, 1024), (1025, 1024)]:
        ms, gbs = run(ctx, W, H, 72)
        print(f"{W}x{H}x72 fused: {ms:.4f} ms  {gbs:.0f} GB/s")
    ms, gbs = run(ctx, 1023, 1024, 72, GL_PATH_GENERIC)
    print(f"1023x1024x72 generic chain: {ms:.4f} ms  {gbs:.0f} GB/s")


if __name__ == "__main__":
    main()
