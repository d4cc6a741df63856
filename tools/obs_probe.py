"""Observation-cycle pieces at 1024^2 x 72: dither on the tensor, the
observation update with host exp (bit-exact default) and with device exp."""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, simple_scan, write_pgm  # noqa: E402


def tm(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * sorted(ts)[n // 2]


def main():
    W, C = 1024, 72
    ctx = g.Context(0)
    occ = make_floorplan(W, W, seed=0)
    m = g.load_map(write_pgm(occ), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    for _ in range(5):
        g.step(t, g.OdometryDelta(0.1, 0.0, 0.02), m, ks, act, ctx)
    f = g.DistanceField(m, ctx)
    js, is_ = np.nonzero(occ == 0)
    a, r = simple_scan(occ, is_[len(is_) // 2] * 0.1 + 0.05, js[len(js) // 2] * 0.1 + 0.05, 0.3)
    scan = g.LidarScan(a, r, 8.0)
    s = g.dither_samples(t, 512)
    print(f"samples {len(s.cells)}")
    print(f"dither(tensor) {tm(lambda: g.dither_samples(t, 512)):.2f} ms")
    for host_exp in (1, 0):
        ctx.set_host_exp(host_exp) if hasattr(ctx, "set_host_exp") else None
        print(f"observation_update host_exp={host_exp}: "
              f"{tm(lambda: g.observation_update(t, s, scan, m, f, g.LikelihoodParams())):.3f} ms")
    print(f"tensor_status (sync) {tm(lambda: g.tensor_status(t)):.3f} ms")


if __name__ == "__main__":
    main()
