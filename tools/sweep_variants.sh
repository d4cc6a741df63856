#!/bin/bash
# Run the smoke check + a short bench for every built fused-kernel variant.
cd "$(dirname "$0")/.."
for d in build/variants/*/; do
  n=$(basename $d)
  r=$(GRIDLOC_B200_LIB=$PWD/$d/libgridloc_b200.so timeout 120 python __graft_entry__.py 2>&1 | tail -1)
  b=$(GRIDLOC_B200_LIB=$PWD/$d/libgridloc_b200.so timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 10 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f Hz  kern %.4f ms  frac %.3f' % (d['value'], d['roofline']['avg_kernel_ms'], d['roofline']['frac']))")
  echo "$n | $r | $b"
done
