# round 2: new parity tests (1000-step default, closed-loop LIDAR, 1024^2x360, concurrency, IPC shards)
# and the tile-order / stack / H=3 rows sweep at c4 and c2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_sharding_ipc.py tests/test_gpu_batch_concurrency.py tests/test_gpu_step_parity.py -q -m gpu > gpurun_out/t_new.log 2>&1; tail -15 gpurun_out/t_new.log
timeout 900 python tools/order_probe.py 4096 4096 360 20 0 16 34 16:4 8:4 4:4 0:4 > gpurun_out/order2_c4.txt 2>&1; cat gpurun_out/order2_c4.txt
timeout 600 python tools/order_probe.py 1024 1024 72 2000 0 0:4 4:4 8:4 > gpurun_out/order2_c2.txt 2>&1; cat gpurun_out/order2_c2.txt
for v in h3r6mb3 h3r5mb3; do GRIDLOC_B200_LIB=$PWD/build/variants/$v/libgridloc_b200.so timeout 900 python tools/order_probe.py 4096 4096 360 20 16 16:4 8:4 > gpurun_out/order2_c4_$v.txt 2>&1; echo $v; cat gpurun_out/order2_c4_$v.txt; done
for o in 16 34 8:4 4:4; do
PASSES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused_step -s 3 -c 1 --csv python tools/order_probe.py 4096 4096 360 1 $o > gpurun_out/ncu2_order_c4_${o/:/_}.csv 2>&1; echo "ncu $o rc=$?"
done
timeout 2400 python -m pytest tests/test_gpu_long_parity.py -q -m gpu > gpurun_out/t_long.log 2>&1; tail -15 gpurun_out/t_long.log
