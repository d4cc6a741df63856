# H=3 tile height at 4 CTAs/SM: 5 and 6 rows vs 4 (parity subset + c4 timing, interleaved)
for v in h3r5mb4 h3r6mb4; do
  GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 900 python -m pytest tests/test_gpu_step_parity.py tests/test_gpu_sharding.py -q -m gpu -x -k "360 or sharded or trace or odd" > gpurun_out/t_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/t_$v.log)"
done
for pass in 1 2; do for v in default h3r5mb4 h3r6mb4; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v pass $pass"; PASSES=1 GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 4096 4096 360 30 -1
done; done > gpurun_out/h3rows.txt 2>&1; cat gpurun_out/h3rows.txt
for v in h3r5mb4; do PASSES=1 GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_fused_step -s 3 -c 1 --csv python tools/order_probe.py 4096 4096 360 1 -1 > gpurun_out/ncu_$v.csv 2>&1; done
grep -E "dram__|gpu__time|fp64" gpurun_out/ncu_h3r5mb4.csv | awk -F'","' '{print $(NF-2), $NF}'
