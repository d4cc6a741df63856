#!/bin/bash
# Run the smoke check + a short bench for every built fused-kernel variant
# (build/variants/<name>/, see build_variants.sh). Extra args go to bench.py,
# e.g. --config c4 --steps 100.
cd "$(dirname "$0")/.."
for d in build/variants/*/; do
  n=$(basename $d)
  r=$(GRIDLOC_B200_LIB=$PWD/$d/libgridloc_b200.so timeout 120 python __graft_entry__.py 2>&1 | tail -1 | cut -c1-40)
  b=$(GRIDLOC_B200_LIB=$PWD/$d/libgridloc_b200.so timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-extras --e2e-steps 10 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f Hz  kern %.4f ms  frac %.3f  sm %s MHz %s' % (d['value'], d['roofline']['avg_kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons']))")
  echo "$n | $r | $b"
done
