# round 2 profiling: benches (c2 sustained, c1, c5), ncu launch list of the default bench command,
# ncu --set full of the fused step at c2 and c4 (strips)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2_full.log 2>&1; tail -1 gpurun_out/bench_c2_full.log | cut -c1-300
for c in c1 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-250; done
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras --e2e-steps 5"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 5 -c 1 -o gpurun_out/r02_prof_c2 $CMD > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
PASSES=1 ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 3 -c 1 -o gpurun_out/r02_prof_c4 python tools/order_probe.py 4096 4096 360 1 -1 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
