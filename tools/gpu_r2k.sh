python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_readouts.py tests/test_gpu_batch_concurrency.py tests/test_gpu_engine.py tests/test_gpu_sharding.py tests/test_gpu_sharding_ipc.py tests/test_gpu_dropin.py -q -m gpu > gpurun_out/t_k.log 2>&1; tail -2 gpurun_out/t_k.log; grep FAILED gpurun_out/t_k.log | head
GRIDLOC_LONG_PARITY=320 timeout 1500 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "closed or devexp" > gpurun_out/t_k2.log 2>&1; tail -2 gpurun_out/t_k2.log
timeout 300 python tools/time_lidar.py > gpurun_out/time_lidar.log 2>&1; tail -1 gpurun_out/time_lidar.log
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-120
