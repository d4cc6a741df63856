# rotated-ring variants: bit-exactness (step parity + sharding subsets) and timing at c4 / c2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for v in rot3 rot1; do
  GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 900 python -m pytest tests/test_gpu_step_parity.py tests/test_gpu_sharding.py tests/test_gpu_engine.py -q -m gpu -x > gpurun_out/t_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/t_$v.log)"
done
timeout 900 python -m pytest tests/test_gpu_seq_sum.py tests/test_gpu_readouts.py tests/test_gpu_engine.py tests/test_gpu_dropin.py -q -m gpu > gpurun_out/t_g.log 2>&1; grep -E "FAILED|passed|failed" gpurun_out/t_g.log | tail -12
for v in default rot3 rot3u2 rot3r6; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v"; GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 4096 4096 360 20 -1
done > gpurun_out/rot_c4.txt 2>&1; cat gpurun_out/rot_c4.txt
for v in default rot1; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v"; GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 1024 1024 72 2000 -1
done > gpurun_out/rot_c2.txt 2>&1; cat gpurun_out/rot_c2.txt
PASSES=1 GRIDLOC_B200_LIB=$PWD/build/variants/rot3/libgridloc_b200.so ncu --set full --clock-control none --import-source on -k regex:k_fused_step -s 3 -c 1 -o gpurun_out/r02_prof_c4_rot3 python tools/order_probe.py 4096 4096 360 1 -1 > gpurun_out/ncu_c4r.log 2>&1; echo "ncu rc=$?"
