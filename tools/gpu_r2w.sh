#!/bin/bash
for r in 1 2; do
for v in pf nopf pfu1; do
  GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 300 python tools/ab_dither.py 1024 40 2>&1 | tail -1
done; done
