mkdir -p gpurun_out/r02u
O=gpurun_out/r02u
timeout 1500 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -k "not full_size and not full_length" > $O/pytest_a.log 2>&1; tail -3 $O/pytest_a.log
timeout 600 python scripts/time_step.py C4 4096 12 2> $O/steps.err | cut -c1-150 > $O/steps.txt; tail -4 $O/steps.txt
timeout 1500 python scripts/long_curve.py C4 4096 120 $O/curve_C4_N4096.json > $O/curve_C4_N4096.log 2>&1; tail -14 $O/curve_C4_N4096.log
