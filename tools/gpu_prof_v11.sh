CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 5 -c 1 -o gpurun_out/prof_v11 $CMD > gpurun_out/ncu.log 2>&1; tail -2 gpurun_out/ncu.log
