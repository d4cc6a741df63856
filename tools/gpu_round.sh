python -m pytest tests/test_gpu_difficulty.py tests/test_gpu_step_parity.py -x -q > gpurun_out/gpu_tests_new.log 2>&1; tail -3 gpurun_out/gpu_tests_new.log
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
