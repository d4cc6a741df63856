CMD="python tools/time_lidar.py 1024"
$CMD > gpurun_out/plain_fs.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_dither_pipe -s 2 -c 1 -o gpurun_out/prof_fs $CMD > gpurun_out/ncu_fs.log 2>&1; tail -2 gpurun_out/ncu_fs.log
