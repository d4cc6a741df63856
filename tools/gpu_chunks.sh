for cfg in c1 c5r; do for c in 0 2 3 4 6 8; do
  echo "$cfg chunks=$c $(GRIDLOC_B200_CHUNKS=$c timeout 300 python bench.py --config $cfg --steps 3000 --warmup 20 --no-cpu-baseline --no-extras --e2e-steps 200 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f Hz kern %.4f ms frac %.3f e2e %.1f Hz' % (d['value'], d['roofline']['avg_kernel_ms'], d['roofline']['frac'], d['e2e']['value']))")"
done; done
