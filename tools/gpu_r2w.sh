#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_seq_sum.py tests/test_gpu_readouts.py tests/test_gpu_engine.py tests/test_gpu_sharding.py tests/test_gpu_dither_seg.py 2>&1 | tail -1
timeout 900 python tools/stress_seqsum.py 1500 2>&1 | tail -1
GRIDLOC_B200_LIB=$PWD/build/variants/dbg/libgridloc_b200.so GL_DEBUG_SEQSUM=1 timeout 300 python tools/argmax_launches.py 2>&1 | grep "seq sum" | tail -2
timeout 300 python tools/time_readouts.py 2>&1 | tail -3
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/argmax_launches2.csv python tools/argmax_launches.py > gpurun_out/argmax.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/argmax_launches2.csv')) if len(r)>10]
h=rows[0]; ci={k:i for i,k in enumerate(h)}
for r in rows[1:]:
    if r[ci['Metric Name']]=='gpu__time_duration.sum':
        print(r[ci['Metric Value']], r[ci['Metric Unit']], r[ci['Kernel Name']][:50])
PY
