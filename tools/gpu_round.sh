# A/B of fused-kernel variants, two passes to see box drift
bash tools/sweep_variants.sh --config c2 > gpurun_out/sweep5a_c2.txt 2>&1; cat gpurun_out/sweep5a_c2.txt
bash tools/sweep_variants.sh --config c2 > gpurun_out/sweep5b_c2.txt 2>&1; cat gpurun_out/sweep5b_c2.txt
bash tools/sweep_variants.sh --config c4 --steps 100 > gpurun_out/sweep5_c4.txt 2>&1; cat gpurun_out/sweep5_c4.txt
