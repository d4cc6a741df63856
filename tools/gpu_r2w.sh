#!/bin/bash
timeout 1500 python -m pytest -q -x tests/test_gpu_step_parity.py tests/test_gpu_readouts.py tests/test_gpu_wall_mask.py tests/test_gpu_sharding.py 2>&1 | tail -2
timeout 300 python tools/time_c3_phases.py 2>&1 | grep "sync=True" | cut -c1-150
timeout 600 python bench.py --steps 2000 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['roofline']['avg_kernel_ms'])"
