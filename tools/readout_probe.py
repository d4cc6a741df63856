"""The read-out and observation kernels at 1024^2x72 (for an ncu launch
list with DRAM bytes: argmax_state incl. the exact sequential total,
belief_map, dither_samples from the tensor, observation_update). Marks the
region of interest with one extra fused step before and after."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, simple_scan, write_pgm  # noqa: E402


def main():
    W, C = 1024, 72
    ctx = g.Context(0)
    occ = make_floorplan(W, W, seed=0)
    m = g.load_map(write_pgm(occ), 250, 0.1, ctx=ctx)
    f = g.DistanceField(m, ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    t = g.init_uniform(m, C, ctx)
    u = g.OdometryDelta(0.1, 0.0, 0.0)
    for _ in range(5):
        g.step(t, u, m, ks, act, ctx)
    js, is_ = np.nonzero(occ == 0)
    q = len(is_) // 2
    a, r = simple_scan(occ, is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.3)
    for _ in range(2):
        g.step(t, u, m, ks, act, ctx)
        est = g.argmax_state(t)
        bm = g.belief_map(t)
        smp = g.dither_samples(t, 512)
        g.observation_update(t, smp, g.LidarScan(a, r, 8.0), m, f, g.LikelihoodParams())
    print(f"argmax ({est.i},{est.j},{est.k}) conf {est.confidence:.6e}; belief map max {bm.max():.3e}; "
          f"{len(smp.cells)} samples")


if __name__ == "__main__":
    main()
