for i in 1 2; do bash tools/sweep_variants.sh; done > gpurun_out/sweep_c2.txt 2>&1; cat gpurun_out/sweep_c2.txt
