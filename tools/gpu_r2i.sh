# TMA stage-count sweep (bytes in flight) at c4 and c2
for v in default ns4 ns5 ns6; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v"; GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 4096 4096 360 20 -1
  GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 1024 1024 72 2000 -1
done > gpurun_out/ns_sweep.txt 2>&1; cat gpurun_out/ns_sweep.txt
for v in default ns5; do
  if [ $v = default ]; then L=$PWD/paper_1910_00572_b200/libgridloc_b200.so; else L=$PWD/build/variants/$v/libgridloc_b200.so; fi
  echo "== $v again"; GRIDLOC_B200_LIB=$L timeout 900 python tools/order_probe.py 4096 4096 360 20 -1
done >> gpurun_out/ns_sweep.txt 2>&1; tail -4 gpurun_out/ns_sweep.txt
