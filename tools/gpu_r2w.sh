#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py 2>&1 | tail -1
timeout 600 python tools/stress_dither.py 1000 2>&1 | tail -1
for r in 1 2; do
for v in base product; do
  if [ $v = product ]; then unset GRIDLOC_B200_LIB; else export GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so; fi
  timeout 300 python tools/ab_dither.py 1024 40 2>&1 | tail -1
done; done; true
