python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_step_parity.py tests/test_gpu_sharding.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -3
for i in 1 2; do bash tools/sweep_variants.sh; done > gpurun_out/sweep_c2.txt 2>&1; cat gpurun_out/sweep_c2.txt
bash tools/sweep_variants.sh --config c4 --steps 100 > gpurun_out/sweep_c4.txt 2>&1; cat gpurun_out/sweep_c4.txt
