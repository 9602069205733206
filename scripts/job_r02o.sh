mkdir -p gpurun_out/r02o
O=gpurun_out/r02o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -k "exact or golden or core_maps or linear_faces or c5_member" > $O/pytest_a.log 2>&1; tail -4 $O/pytest_a.log
timeout 600 python scripts/time_step.py C4 4096 12 2> $O/steps.err | cut -c1-150 > $O/steps.txt; tail -5 $O/steps.txt
timeout 600 python scripts/timeline.py C4 4096 8 > $O/timeline.txt 2>&1; tail -40 $O/timeline.txt
