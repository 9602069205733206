set -x
timeout 1200 python -m pytest tests -q -m gpu --durations=5 -x -k "not c3_small" > gpurun_out/pytest_gpu.log 2>&1; tail -8 gpurun_out/pytest_gpu.log
timeout 300 python scripts/time_step.py C1 256 4 | tail -2
timeout 300 python scripts/time_step.py C2 1024 4 | tail -2
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v2c.json 2> gpurun_out/bench_v2c.err; cat gpurun_out/bench_v2c.json; tail -3 gpurun_out/bench_v2c.err
