#!/usr/bin/env python
"""Randomised stress of the exact sequential sum against the literal chain
(validation tool): random lengths (1 .. 400K), exponent ranges, zero runs,
ties and signed zeros."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402


def seq(x):
    t = 0.0
    for v in x.tolist():
        t += v
    return t


def draw(rng):
    n = int(rng.choice([1, 7, 100, 8191, 8192, 8193, 16384 + 5, int(rng.integers(1, 400_000))]))
    lo, hi = sorted(rng.uniform(-300, 300, 2))
    kind = int(rng.integers(0, 5))
    if kind == 0:
        x = 10.0 ** rng.uniform(lo, hi, n)
    elif kind == 1:  # growing: crossings
        x = 2.0 ** np.linspace(lo * 3.3, hi * 3.3, n) * rng.random(n)
    elif kind == 2:  # ties at one scale after a big head
        e = int(rng.integers(-60, 0))
        x = np.concatenate([[2.0 ** (e + 53)], rng.integers(0, 4, n) * 2.0 ** (e - 1)])
    elif kind == 3:  # zero runs and -0.0
        x = np.where(rng.random(n) < 0.7, 0.0, rng.random(n) * 10.0 ** rng.uniform(lo, hi))
        x[rng.random(n) < 0.05] = -0.0
    else:  # subnormals into normals
        x = np.concatenate([rng.integers(0, 9, n) * 5e-324, rng.random(n // 3 + 1)])
    return np.ascontiguousarray(x, dtype=np.float64)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    ctx = g.Context(0)
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 777)
    bad = 0
    for i in range(n):
        x = draw(rng)
        got, want = g.sequential_sum(x, ctx), seq(x)
        if np.float64(got).view(np.uint64) != np.float64(want).view(np.uint64):
            bad += 1
            print("MISMATCH", i, x.size, got, want)
    print(f"{n} cases, {bad} mismatches")


if __name__ == "__main__":
    main()
