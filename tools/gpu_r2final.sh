#!/bin/bash
# full GPU suite + smoke + every bench config + the reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log; grep FAILED gpurun_out/t_all.log | head -20
for c in c2 c3 c1 c5 c4; do
  steps=""; [ $c = c4 ] && steps="--steps 100"
  timeout 900 python bench.py --config $c $steps > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-160
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
