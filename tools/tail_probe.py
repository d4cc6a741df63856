"""Does the fused step's time follow the number of tile waves? Time the
1024-wide step at heights around the 2-wave boundary (4736 warp tiles at
16 warps/SM x 148 SMs = 2 waves = 135.3 tile rows of 8)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm  # noqa: E402


def main():
    ctx = g.Context(0)
    C = 72
    for H in [960, 1000, 1024, 1048, 1072, 1080, 1088, 1104]:
        occ = make_floorplan(1024, H, seed=0)
        m = g.load_map(write_pgm(occ), 250, 0.1, ctx=ctx)
        ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
        act = g.make_activation(m, ks, C, ctx)
        t = g.init_uniform(m, C, ctx)
        u = g.OdometryDelta(0.1, 0.0, 0.0)
        for _ in range(20):
            g.step_async(t, u, m, ks, act, ctx)
        ctx.synchronize()
        ctx.mark(0)
        n = 400
        for _ in range(n):
            g.step_async(t, u, m, ks, act, ctx)
        ctx.mark(1)
        ctx.synchronize()
        ms = ctx.marks_ms(0, 1) / n
        tiles = 35 * math.ceil(H / 8)
        print(f"H={H} tiles={tiles} waves={tiles / 2368:.3f} ms/step={ms:.4f} us/tile-row={1000 * ms / math.ceil(H / 8):.3f}")
        del t, act, ks, m


if __name__ == "__main__":
    main()
