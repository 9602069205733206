timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_v8b.log 2>&1
