mkdir -p gpurun_out/r02w
O=gpurun_out/r02w
TTSW_LONG_FULL=1 timeout 5000 python -m pytest tests/test_gpu_long.py -q --durations=10 -k "c5_m1 or c5_m5" > $O/pytest_long.log 2>&1; tail -8 $O/pytest_long.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/
