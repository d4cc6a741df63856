#!/usr/bin/env python
"""GPU dither vs the C oracle on a random (W, W) plane (usage: W)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1910_00572_b200 as g
from oracle import Port
W = int(sys.argv[1])
rng = np.random.default_rng(1)
bm = rng.random((W, W)) ** 8
bm[rng.random((W, W)) < 0.3] = 0.0
ctx = g.Context(0)
s = g.dither_samples(bm, 512, ctx)
p = Port()
cells, mass = p.dither(bm, 512)
print(W, len(s.cells), len(cells), s.source_mass == mass, np.array_equal(s.cells, cells))
