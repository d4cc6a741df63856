#!/bin/bash
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_dither_seg -c 1 -o gpurun_out/dither_seg -f python tools/obs_cycle.py 160 > gpurun_out/dither_seg.log 2>&1
tail -1 gpurun_out/dither_seg.log
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-200
