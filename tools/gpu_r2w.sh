#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py 2>&1 | tail -1
timeout 600 python tools/stress_dither.py 2000 2>&1 | tail -1
for v in base product; do
  if [ $v = product ]; then unset GRIDLOC_B200_LIB; else export GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so; fi
  timeout 600 python tools/late_dither.py 400 800 1600 2400 2>&1 | tail -4
  timeout 300 python tools/ab_dither.py 1024 20 2>&1 | tail -1 | cut -c1-60
done; true
