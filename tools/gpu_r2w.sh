#!/bin/bash
for r in 1 2; do
for v in base product; do
  if [ $v = product ]; then unset GRIDLOC_B200_LIB; else export GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so; fi
  timeout 300 python tools/ab_dither.py 1024 40 2>&1 | tail -1
  [ $r = 1 ] && timeout 300 python tools/time_c3_phases.py 2>&1 | grep "sync=True" | cut -c1-120
done; done; true
