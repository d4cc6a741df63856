#!/bin/bash
for v in at1 at4 product; do
  if [ $v = product ]; then unset GRIDLOC_B200_LIB; else export GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so; fi
  timeout 600 python tools/late_dither.py 400 800 1600 2400 2>&1 | tail -4
  timeout 300 python tools/ab_dither.py 1024 20 2>&1 | tail -1 | cut -c1-60
done; true
