python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py tests/test_gpu_seq_sum.py -q -m gpu > gpurun_out/t_q.log 2>&1; tail -2 gpurun_out/t_q.log; grep FAILED gpurun_out/t_q.log | head -20
timeout 300 python tools/time_lidar.py > gpurun_out/time_lidar.log 2>&1; tail -1 gpurun_out/time_lidar.log
GRIDLOC_LONG_PARITY=320 timeout 1500 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "closed" > gpurun_out/t_q2.log 2>&1; tail -2 gpurun_out/t_q2.log
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-120
