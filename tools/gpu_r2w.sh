#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_readouts.py tests/test_gpu_batch_concurrency.py 2>&1 | tail -1
timeout 600 python bench.py --config c5 --steps 1000 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5',d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
