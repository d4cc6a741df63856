#!/bin/bash
timeout 1200 python -m pytest -q -x tests/test_gpu_seq_sum.py tests/test_gpu_readouts.py tests/test_gpu_engine.py tests/test_gpu_sharding.py tests/test_gpu_sharding_ipc.py tests/test_gpu_dropin.py tests/test_gpu_dither_seg.py 2>&1 | tail -2
timeout 300 python tools/time_readouts.py 2>&1 | tail -3
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/argmax_launches.csv python tools/argmax_launches.py > gpurun_out/argmax.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/argmax_launches.csv')) if len(r)>10]
h=rows[0]; ci={k:i for i,k in enumerate(h)}
tot=0
for r in rows[1:]:
    if r[ci['Metric Name']]=='gpu__time_duration.sum':
        print(r[ci['Metric Value']], r[ci['Metric Unit']], r[ci['Kernel Name']][:70]); tot+=float(r[ci['Metric Value']])
print('total', tot)
PY
