#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_seq_sum.py 2>&1 | tail -2
