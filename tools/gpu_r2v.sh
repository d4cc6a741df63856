#!/bin/bash
GRIDLOC_B200_LIB=$PWD/build/variants/dbg/libgridloc_b200.so GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py 2>&1 | tail -2
