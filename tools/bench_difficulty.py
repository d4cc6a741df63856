"""map_difficulty (evaluation.cpp:25-72): device vs the reference's CPU
implementation (oracle/_ref, all host threads), default DifficultyConfig,
on the reference's fixed worlds and a strided floor plan. Prints one JSON
line per map: seconds, candidates/s and whether the fractions are equal."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (the checker and CPU baseline, not the product)
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan  # noqa: E402

ref = oracle.Ref()
ctx = g.Context(0)
cases = [(f"world{w}", oracle.ref_world_cells(ref, w), 1) for w in range(4)]
cases.append(("floor256_stride2", make_floorplan(256, 256, seed=0), 2))
for name, occ, stride in cases:
    h, w = occ.shape
    m = g.OccupancyMap(w, h, 0.1, occ, ctx=ctx)
    f = g.DistanceField(m, ctx)
    cfg = g.DifficultyConfig(stride=stride)
    g.map_difficulty(m, f, cfg, ctx)  # warm-up (tables, allocation)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        ours = g.map_difficulty(m, f, cfg, ctx)
        ts.append(time.perf_counter() - t0)
    gpu_s = sorted(ts)[1]
    rm = oracle.RefMap(ref, occ=occ)
    rcfg = dict(thr=1.0, beams=8, fov=2 * math.pi, max_range=8.0, stride=stride, bins=8, lik=(0.2, 0.05, 1))
    t0 = time.perf_counter()
    theirs = oracle.ref_map_difficulty(ref, rm, rcfg)
    cpu_s = time.perf_counter() - t0
    n = sum(1 for j in range(1, h - 1, stride) for i in range(1, w - 1, stride) if occ[j, i] == 0)
    cands = n * n * 8
    print(json.dumps({"map": name, "W": w, "H": h, "stride": stride, "query_cells": n,
                      "likelihoods": cands, "gpu_s": gpu_s, "cpu_s": cpu_s, "cpu_threads": os.cpu_count(),
                      "speedup": cpu_s / gpu_s, "gpu_likelihoods_per_s": cands / gpu_s,
                      "fraction": ours, "equal": ours == theirs}), flush=True)
