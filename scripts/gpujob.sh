set -x
timeout 1200 python -m pytest tests -q -m gpu -x -k "not c3_small" --durations=6 > gpurun_out/pytest_gpu.log 2>&1; tail -12 gpurun_out/pytest_gpu.log
timeout 300 python scripts/time_step.py C2 1024 3 | tail -1
timeout 900 python scripts/time_step.py C3 512 2 | tail -2
