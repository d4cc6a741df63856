python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/t_full.log 2>&1; tail -3 gpurun_out/t_full.log; grep FAILED gpurun_out/t_full.log | head
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_drv.log 2>&1; tail -1 gpurun_out/bench_drv.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
