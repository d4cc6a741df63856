# final validation of the wave-tail default: smoke, all GPU tests, benches, ncu launch list + full capture
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
for c in c3 c5 c1; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-160; done
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 5"
$CMD > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv --log-file gpurun_out/launches_tail.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 5 -c 1 -o gpurun_out/prof_tail $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu.log
