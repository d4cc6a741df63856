#!/usr/bin/env python
"""A/B timing of the dither sweep (experiment only): the dither of a
1024^2x72 belief tensor, CUDA-event timed on the context stream, median and
min of N runs, for whichever library GRIDLOC_B200_LIB points at."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    C = 72
    ctx = g.Context(0)
    occ = make_floorplan(W, W, seed=0)
    m = g.load_map(write_pgm(occ), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    tt = g.init_uniform(m, C, ctx)
    for _ in range(5):
        g.step(tt, g.OdometryDelta(0.1, 0.0, 0.02), m, ks, act, ctx)
    import time
    g.dither_samples(tt, 512)
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        s = g.dither_samples(tt, 512)
        ts.append(1e3 * (time.perf_counter() - t0))
    bm = g.belief_map(tt)
    tb = []
    for _ in range(n):
        t0 = time.perf_counter()
        g.belief_map(tt)
        tb.append(1e3 * (time.perf_counter() - t0))
    lib = os.environ.get("GRIDLOC_B200_LIB", "product")
    print(f"{os.path.basename(os.path.dirname(lib)) or lib}: dither(tensor) median {np.median(ts):.3f} min {min(ts):.3f} ms; "
          f"belief_map median {np.median(tb):.3f} ms; samples {len(s.cells)} hash {hash(tuple(map(tuple, np.asarray(s.cells).tolist())))}")


if __name__ == "__main__":
    main()
