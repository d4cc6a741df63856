#!/bin/bash
timeout 1200 python -m pytest -q -x tests/test_gpu_seq_sum.py tests/test_gpu_readouts.py tests/test_gpu_dither_seg.py tests/test_gpu_engine.py tests/test_gpu_sharding.py tests/test_gpu_dropin.py 2>&1 | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/obs_cycle_launches5.csv python tools/obs_cycle.py 160 > gpurun_out/obs_cycle.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/obs_cycle_launches5.csv')) if len(r)>10]
h=rows[0]; ci={k:i for i,k in enumerate(h)}
tot=0
for r in rows[1:]:
    if r[ci['Metric Name']]=='gpu__time_duration.sum':
        v=float(r[ci['Metric Value']]); tot+=v
        print(r[ci['Metric Value']], r[ci['Metric Unit']], r[ci['Kernel Name']][:60])
print('total', tot)
PY
timeout 300 python tools/time_c3_phases.py 2>&1 | grep "sync=True" | cut -c1-150
