#!/bin/bash
# dither sweep check: parity subset + phase clocks + lidar timing + the c3 loop phases
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_dither_wide.py tests/test_gpu_readouts.py 2>&1 | tail -3
GRIDLOC_B200_LIB=$PWD/build/variants/dbg/libgridloc_b200.so GL_DEBUG_DITHER=1 timeout 300 python tools/time_c3_phases.py 2>&1 | grep -E "dither (clocks|events)|Hz" | awk 'NR%4==1 || /Hz/' | cut -c1-200 | head -40
timeout 300 python tools/time_c3_phases.py 2>&1 | tail -4
