mkdir -p gpurun_out/r02v
O=gpurun_out/r02v
timeout 3000 python -m pytest tests/test_gpu_long.py -q --durations=10 -k "c5_m0 or c5_m1 or c5_m2 or c4_n4096" > $O/pytest_long.log 2>&1; tail -25 $O/pytest_long.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/
