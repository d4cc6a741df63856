python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_readouts.py tests/test_gpu_batch_concurrency.py tests/test_gpu_engine.py tests/test_gpu_sharding.py tests/test_gpu_dropin.py tests/test_gpu_seq_sum.py -q -m gpu > gpurun_out/t_j.log 2>&1; tail -2 gpurun_out/t_j.log; grep FAILED gpurun_out/t_j.log | head
GL_DEBUG_DITHER=0 timeout 300 python tools/time_lidar.py > gpurun_out/time_lidar.log 2>&1; tail -2 gpurun_out/time_lidar.log
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-120
