"""Generate the recorded odometry-trace fixtures used by bench.py's
recorded-trace stream and by parity tests that must not depend on the
reference at run time.

The reference simulator (RandomWalkPolicy, step_robot, odometry_measurement;
simulator.cpp) and the Localizer trigger (localizer.cpp:25-46) run through
the compiled reference (oracle/_ref) on the floor plan the bench uses; every
step() the Localizer would issue is recorded as (u, v, w, slot) with slot 0 =
main kernels, 1 = rotation-only kernels.

  python tests/golden/make_traces.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan  # noqa: E402

SPECS = [  # (name, W, H, channels, map seed, trace seed, steps)
    ("trace_1024x72", 1024, 1024, 72, 0, 11, 2000),
    ("trace_256x36", 256, 256, 36, 0, 3, 1000),
    ("trace_4096x360", 4096, 4096, 360, 0, 7, 500),
]


def main():
    ref = oracle.Ref()
    for name, W, H, C, mseed, tseed, n in SPECS:
        occ = make_floorplan(W, H, seed=mseed)
        rm = oracle.RefMap(ref, occ=occ)
        js, is_ = np.nonzero(occ == 0)
        q = len(is_) // 3
        start = (is_[q] * 0.1 + 0.05, js[q] * 0.1 + 0.05, 0.5)
        ev, _ = oracle.ref_gen_trace(ref, rm, C, start, seed=tseed, max_steps=n)
        steps = ev[ev[:, 0] == 0][:, 1:5].copy()
        np.save(os.path.join(HERE, name + ".npy"), steps)
        print(name, steps.shape, "rotation-only share", float(steps[:, 3].mean()))


if __name__ == "__main__":
    main()
