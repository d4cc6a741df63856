python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_wall_mask.py tests/test_gpu_engine.py tests/test_gpu_dropin.py tests/test_gpu_raycast.py tests/test_gpu_dither_wide.py -q -m gpu > gpurun_out/t_d.log 2>&1; tail -40 gpurun_out/t_d.log
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_long_parity.py > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
