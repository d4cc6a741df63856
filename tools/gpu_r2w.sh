#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py 2>&1 | tail -2
GRIDLOC_B200_LIB=$PWD/build/variants/dbg/libgridloc_b200.so GL_DEBUG_DITHER=1 timeout 300 python tools/ab_dither.py 1024 3 2>&1 | grep -E "dither (clocks|events)" | tail -2
timeout 300 python tools/ab_dither.py 1024 40 2>&1 | tail -1
timeout 300 python tools/time_c3_phases.py 2>&1 | grep "sync=True" | cut -c1-150
