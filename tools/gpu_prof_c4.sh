CMD="python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1"
$CMD > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 3 -c 1 -o gpurun_out/prof_c4_stack $CMD > gpurun_out/ncu_c4.log 2>&1; tail -2 gpurun_out/ncu_c4.log
