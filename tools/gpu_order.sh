# round 2: tile-order (strip) sweep at c4 / c2, the H=3 6-row variant, and dram bytes per order under ncu
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python tools/order_probe.py 4096 4096 360 20 0 4 8 16 34 > gpurun_out/order_c4.txt 2>&1; cat gpurun_out/order_c4.txt
timeout 600 python tools/order_probe.py 1024 1024 72 2000 0 2 4 8 > gpurun_out/order_c2.txt 2>&1; cat gpurun_out/order_c2.txt
GRIDLOC_B200_LIB=$PWD/build/variants/h3r6mb3/libgridloc_b200.so timeout 900 python tools/order_probe.py 4096 4096 360 20 0 8 16 > gpurun_out/order_c4_h3r6.txt 2>&1; cat gpurun_out/order_c4_h3r6.txt
for o in 0 8; do
PASSES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_fused_step -s 3 -c 1 --csv python tools/order_probe.py 4096 4096 360 1 $o > gpurun_out/ncu_order_c4_$o.csv 2>&1; echo "ncu $o rc=$?"
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
