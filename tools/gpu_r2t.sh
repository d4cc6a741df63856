#!/bin/bash
# dither sweep check: parity subset + phase clocks + lidar timing
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_dither_wide.py tests/test_gpu_readouts.py 2>&1 | tail -3
GRIDLOC_B200_LIB=$PWD/build/variants/dbg/libgridloc_b200.so GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py 2>&1 | tail -4
timeout 300 python tools/time_lidar.py 2>&1 | tail -3
