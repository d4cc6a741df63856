#!/bin/bash
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_dither_seg -c 1 -o gpurun_out/dither_seg -f python tools/obs_cycle.py 160 > gpurun_out/dither_seg.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:k_dither_seg -c 1 -o gpurun_out/dither_seg_early -f python tools/obs_cycle.py 16 > gpurun_out/dither_seg_early.log 2>&1
tail -1 gpurun_out/dither_seg.log; tail -1 gpurun_out/dither_seg_early.log
