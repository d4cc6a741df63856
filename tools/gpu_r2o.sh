# H<=1 tile height 9 / 10 rows at 4 CTAs/SM vs 8: parity subset + c2 timing (interleaved) + c5 batch
for v in h1r9 h1r10; do
  GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 900 python -m pytest tests/test_gpu_step_parity.py -q -m gpu -x > gpurun_out/t_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/t_$v.log)"
done
for pass in 1 2 3; do for v in default h1r9 h1r10; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v pass $pass"; PASSES=1 GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 1024 1024 72 3000 -1
done; done > gpurun_out/h1rows.txt 2>&1; cat gpurun_out/h1rows.txt
for v in default h1r10; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v c5"; GRIDLOC_B200_LIB=$L timeout 600 python bench.py --config c5 --steps 1000 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-160
  echo "== $v c1"; GRIDLOC_B200_LIB=$L timeout 600 python bench.py --config c1 --steps 3000 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | cut -c1-160
done
