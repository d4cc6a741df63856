python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_long_parity.py > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log; grep FAILED gpurun_out/t_all.log | head
timeout 2400 python -m pytest tests/test_gpu_long_parity.py -q -m gpu > gpurun_out/t_long.log 2>&1; tail -3 gpurun_out/t_long.log
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-200
