mkdir -p gpurun_out/r02x
O=gpurun_out/r02x
TTSW_LONG_FULL=1 timeout 6000 python -m pytest tests/test_gpu_long.py -q --durations=10 -k "c3_n32 or c4_n32" > $O/pytest_long.log 2>&1; tail -8 $O/pytest_long.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/
