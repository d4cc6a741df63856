#!/bin/bash
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3_400.log 2>&1; tail -1 gpurun_out/bench_c3_400.log | cut -c1-120
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/obs_cycle_launches6.csv python tools/obs_cycle.py 160 > gpurun_out/obs_cycle.log 2>&1; tail -1 gpurun_out/obs_cycle.log
