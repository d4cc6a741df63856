#!/bin/bash
for r in 1 2; do
for v in base hm; do
  echo "== $v"
  GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 300 python tools/ab_dither.py 1024 40 2>&1 | tail -1
  GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 300 python tools/time_c3_phases.py 2>&1 | grep "sync=True" | cut -c1-140
done; done
