# one gpurun call: parity tests, then the headline bench lines
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-300
python bench.py --config c4 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-200
python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log | cut -c1-200
python bench.py --config c2 --shard --steps 1000 --warmup 10 > gpurun_out/bench_shard_c2.log 2>&1; tail -1 gpurun_out/bench_shard_c2.log | cut -c1-200
python bench.py --config c4 --shard --steps 100 --warmup 5 > gpurun_out/bench_shard_c4.log 2>&1; tail -1 gpurun_out/bench_shard_c4.log | cut -c1-200
