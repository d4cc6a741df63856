CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 5"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_l.log 2>&1; tail -1 gpurun_out/ncu_l.log | cut -c1-200
