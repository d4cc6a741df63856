GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py 1024 > gpurun_out/time_lidar.txt 2>&1; cat gpurun_out/time_lidar.txt | tail -8
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 5"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches_v10.csv $CMD > gpurun_out/ncu_l.log 2>&1; tail -2 gpurun_out/ncu_l.log
