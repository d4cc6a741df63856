#!/bin/bash
GRIDLOC_B200_LIB=$PWD/build/variants/few16/libgridloc_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py 2>&1 | tail -1
for v in few16 few24 product; do
  if [ $v = product ]; then unset GRIDLOC_B200_LIB; else export GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so; fi
  timeout 600 python tools/late_dither.py 400 800 1600 2400 2>&1 | tail -4
done; true
