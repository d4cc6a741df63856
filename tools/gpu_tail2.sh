# wave-tail split, second sweep (GRIDLOC_B200_TAIL="ctas,chunks"): c2 fine grid, c4 check, new-build parity
timeout 900 python -m pytest tests/test_gpu_step_parity.py -x -q -k wave_tail > gpurun_out/tail2_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/tail2_parity.log
one() {  # cfg steps tail
  GRIDLOC_B200_TAIL=$3 timeout 300 python bench.py --config $1 --steps $2 --warmup 10 --no-cpu-baseline --no-extras --e2e-steps 20 > gpurun_out/tail_b.log 2>&1
  python - "$1 $3" <<'PY'
import json,sys
l=open("gpurun_out/tail_b.log").read().strip().splitlines()[-1]
try:
    d=json.loads(l); print(sys.argv[1], "kernel_ms %.4f" % d["roofline"]["avg_kernel_ms"], "Hz %.1f" % d["value"], "frac %.3f" % d["roofline"]["frac"], "mhz", d["clocks"]["sm_mhz"])
except Exception as e: print(sys.argv[1], "ERR", l[:300])
PY
}
for rep in 1 2; do
for t in 0 64,3 96,3 128,3 160,3 128,4 192,4 132,3 0; do one c2 3000 $t; done
for t in 0 92,3 184,3; do one c4 60 $t; done
done
