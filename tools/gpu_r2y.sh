#!/bin/bash
# full GPU suite + smoke + c2/c3 bench lines
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log; grep FAILED gpurun_out/t_all.log | head -20
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
