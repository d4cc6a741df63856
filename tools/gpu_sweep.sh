# variant sweep: c2 twice over every variant, then c4 once
for i in 1 2; do bash tools/sweep_variants.sh; done > gpurun_out/sweep_c2.txt 2>&1; cat gpurun_out/sweep_c2.txt
bash tools/sweep_variants.sh --config c4 --steps 100 > gpurun_out/sweep_c4.txt 2>&1; cat gpurun_out/sweep_c4.txt
