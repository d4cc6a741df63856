#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_gpu_dither_seg.py tests/test_gpu_readouts.py tests/test_gpu_seq_sum.py tests/test_gpu_bench_contract.py 2>&1 | tail -1
timeout 600 python bench.py 2>&1 | tail -1 | cut -c1-300
