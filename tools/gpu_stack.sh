for i in 1 2; do bash tools/sweep_variants.sh --config c4 --steps 100; done > gpurun_out/s4.txt 2>&1; cat gpurun_out/s4.txt
bash tools/sweep_variants.sh > gpurun_out/s2.txt 2>&1; cat gpurun_out/s2.txt
