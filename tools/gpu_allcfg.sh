# one bench line per config (default flags) into gpurun_out/bench_<cfg>.json
for cfg in c2 c3 c1 c5 c4; do
  timeout 900 python bench.py --config $cfg $( [ $cfg = c4 ] && echo "--steps 200 --e2e-steps 20" ) > gpurun_out/bench_$cfg.log 2>&1
  tail -1 gpurun_out/bench_$cfg.log > gpurun_out/bench_$cfg.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$cfg.json')); r=d.get('roofline') or {}; print('$cfg', round(d['value'],1), d['unit'], 'frac', r.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), d['clocks'])"
done
