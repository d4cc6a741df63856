#!/bin/bash
GRIDLOC_B200_LIB=$PWD/build/variants/dbg/libgridloc_b200.so GL_DEBUG_DITHER=1 timeout 300 python tools/time_c3_phases.py 2>&1 | grep -E "dither (clocks|events)|Hz" | awk 'NR%4==1 || /Hz/' | head -80
