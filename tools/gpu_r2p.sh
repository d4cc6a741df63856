python tools/readout_probe.py > gpurun_out/readout_plain.log 2>&1; tail -1 gpurun_out/readout_plain.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_readout_launches.csv python tools/readout_probe.py > gpurun_out/ncu_readout.log 2>&1; echo "ncu rc=$?"
