#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_dither_wide.py 2>&1 | tail -1
timeout 600 python tools/stress_dither.py 2000 2>&1 | tail -1
timeout 600 python tools/late_dither.py 400 800 1600 2400 2>&1 | tail -4
timeout 900 python bench.py --config c3 --steps 3000 --warmup 20 --no-cpu-baseline --no-extras 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3',d['value'],d['e2e']['value'],d['extras'])"
