#!/bin/bash
timeout 1500 python -m pytest -q -x tests/test_gpu_step_parity.py tests/test_capi.py tests/test_gpu_long_parity.py -k "not lidar and not 360" 2>&1 | tail -2
timeout 300 python tools/host_probe.py 2>&1 | tail -1
timeout 300 python tools/host_probe.py 1024 72 2>&1 | tail -1
for c in c1 c2; do
timeout 600 python bench.py --config $c --steps 2000 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c',d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done
