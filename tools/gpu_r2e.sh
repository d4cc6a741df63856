python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_seq_sum.py tests/test_gpu_wall_mask.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py -q -m gpu > gpurun_out/t_e.log 2>&1; grep -E "FAILED|passed|failed" gpurun_out/t_e.log | tail -20
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-600
GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py > gpurun_out/time_lidar.log 2>&1; tail -8 gpurun_out/time_lidar.log
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_long_parity.py > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
