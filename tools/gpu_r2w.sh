#!/bin/bash
timeout 1500 python -m pytest -q -x tests/test_gpu_step_parity.py tests/test_gpu_readouts.py tests/test_gpu_engine.py tests/test_gpu_batch_concurrency.py tests/test_gpu_dropin.py tests/test_gpu_sharding_ipc.py 2>&1 | tail -2
for c in c1 c2; do
timeout 600 python bench.py --config $c --steps 2000 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c',d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done
