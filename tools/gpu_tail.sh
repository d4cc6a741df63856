# wave-tail split sweep (GRIDLOC_B200_TAIL="ctas,chunks") on c2 + parity of the tail path
for t in 5,2 100000,3; do
  GRIDLOC_B200_TAIL=$t timeout 600 python -m pytest tests/test_gpu_step_parity.py -x -q > gpurun_out/tail_parity_$t.log 2>&1; echo "parity tail=$t rc=$?"; tail -1 gpurun_out/tail_parity_$t.log
done
for rep in 1 2; do
for t in 0 64 128 192 264 400 528 128,3 264,3 528,3; do
  GRIDLOC_B200_TAIL=$t timeout 300 python bench.py --steps 3000 --warmup 20 --no-cpu-baseline --no-extras --e2e-steps 50 > gpurun_out/tail_b.log 2>&1
  python - "$t" <<'PY'
import json,sys
l=open("gpurun_out/tail_b.log").read().strip().splitlines()[-1]
try:
    d=json.loads(l); print("tail", sys.argv[1], "kernel_ms %.4f" % d["roofline"]["avg_kernel_ms"], "Hz %.0f" % d["value"], "frac %.3f" % d["roofline"]["frac"], "mhz", d["clocks"]["sm_mhz"])
except Exception as e: print("tail", sys.argv[1], "ERR", l[:300])
PY
done; done
