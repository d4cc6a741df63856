# round 2: wall mask, engine, dropin (incl. sharded localizer), full GPU suite, c2/c4 bench lines
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_wall_mask.py tests/test_gpu_engine.py tests/test_gpu_dropin.py -q -m gpu -x > gpurun_out/t_c.log 2>&1; tail -25 gpurun_out/t_c.log
timeout 600 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
timeout 900 python bench.py --config c4 --steps 60 --warmup 5 --e2e-steps 10 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log
timeout 300 python bench.py --gpus 2 --steps 5 > gpurun_out/bench_g2.log 2>&1; echo "gpus2 rc=$?"; tail -2 gpurun_out/bench_g2.log
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_long_parity.py > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
