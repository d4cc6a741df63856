#!/usr/bin/env python
"""Randomised stress of dither_samples against the oracle (experiment /
validation tool): random widths, heights, plane kinds and budgets."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1910_00572_b200 as g  # noqa: E402
from tests.test_gpu_dither_seg import _plane  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    ctx = g.Context(0)
    port = oracle.Port()
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
    kinds = ["sparse", "dense", "blobs", "walls", "spikes", "tails"]
    bad = 0
    for i in range(n):
        w = int(rng.integers(200, 6400)) if rng.random() < 0.3 else int(rng.integers(200, 1500))
        h = int(rng.integers(1, 60))
        kind = kinds[i % len(kinds)]
        budget = int(rng.choice([16, 512, 4096, 100000]))
        bm = _plane(kind, w, h, int(rng.integers(1 << 30)))
        if rng.random() < 0.2:  # exact zero rows / columns
            bm[rng.integers(0, h, 3), :] = 0.0
        s = g.dither_samples(bm, budget, ctx)
        cells, mass = port.dither(bm, budget)
        ok = s.source_mass == mass and np.array_equal(s.cells, cells)
        if not ok:
            bad += 1
            print("MISMATCH", i, kind, w, h, budget, len(s.cells), len(cells))
    print(f"{n} cases, {bad} mismatches")


if __name__ == "__main__":
    main()
