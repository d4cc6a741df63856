#!/bin/bash
# the final validation: full GPU suite, every bench config, the reference arm, and the 3000-step closed loop
bash tools/gpu_r2final.sh
GRIDLOC_LONG_PARITY=3000 timeout 2000 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k closed > gpurun_out/t_closed3000.log 2>&1; tail -1 gpurun_out/t_closed3000.log
