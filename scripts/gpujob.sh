set -x
timeout 1200 python -m pytest tests -q -m gpu --durations=8 -x > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err; cat gpurun_out/bench_v2.json; tail -3 gpurun_out/bench_v2.err
timeout 300 python scripts/time_step.py C1 256 4 | tail -2
timeout 300 python scripts/time_step.py C3 256 2 | tail -2
