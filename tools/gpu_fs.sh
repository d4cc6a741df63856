timeout 600 python -m pytest tests/test_gpu_readouts.py tests/test_gpu_long_parity.py -x -q 2>&1 | tail -3
GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py 1024 2>&1 | tail -2
GL_DEBUG_DITHER=1 timeout 300 python tools/time_lidar.py 2048 2>&1 | tail -2
