for v in fs2 fs3; do echo "== $v"; GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py 2>&1 | tail -3; done > gpurun_out/fs_var.txt; cat gpurun_out/fs_var.txt
timeout 1500 python -m pytest tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py tests/test_gpu_seq_sum.py tests/test_gpu_batch_concurrency.py -q -m gpu > gpurun_out/t_m.log 2>&1; tail -2 gpurun_out/t_m.log
GRIDLOC_LONG_PARITY=320 timeout 1500 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "closed" > gpurun_out/t_m2.log 2>&1; tail -2 gpurun_out/t_m2.log
timeout 600 python bench.py --config c3 --steps 400 --warmup 20 > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-120
