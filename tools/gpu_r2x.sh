#!/bin/bash
# ncu source-level capture of the segment sweep (one launch)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_dither_seg -c 1 \
  -o gpurun_out/seg_src -f python tools/ab_dither.py 1024 2 > gpurun_out/seg_src.log 2>&1
tail -3 gpurun_out/seg_src.log
