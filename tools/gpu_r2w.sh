#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_bench_contract.py tests/test_capi.py 2>&1 | tail -1
for c in c1 c2 c5; do
timeout 600 python bench.py --config $c --steps 2000 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c',d['value'],d['e2e']['value'],d['roofline']['frac'],d['roofline'].get('launches_timed'),d['clocks']['sm_mhz'])"
done
