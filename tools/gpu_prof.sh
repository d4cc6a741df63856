# c1 chunk sweep (plain), then one ncu --set full capture of the c2 fused step
for c in 0 1 2 4 9 18; do
  echo "chunks=$c $(GRIDLOC_B200_CHUNKS=$c timeout 300 python bench.py --config c1 --steps 3000 --warmup 20 --no-cpu-baseline --no-extras --e2e-steps 200 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f Hz kern %.4f ms e2e %.1f Hz' % (d['value'], d['roofline']['avg_kernel_ms'], d['e2e']['value']))")"
done > gpurun_out/c1_chunks.txt 2>&1; cat gpurun_out/c1_chunks.txt
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 5 -c 1 -o gpurun_out/prof_v10 $CMD > gpurun_out/ncu.log 2>&1; tail -3 gpurun_out/ncu.log
