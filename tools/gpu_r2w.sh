#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py 2>&1 | tail -2
GRIDLOC_B200_LIB=$PWD/build/variants/cw1/libgridloc_b200.so timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py 2>&1 | tail -1
for v in cw1 product; do
  if [ $v = product ]; then unset GRIDLOC_B200_LIB; else export GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so; fi
  timeout 300 python tools/ab_dither.py 1024 40 2>&1 | tail -1
  timeout 300 python tools/time_c3_phases.py 2>&1 | grep "sync=True" | cut -c1-150
done
