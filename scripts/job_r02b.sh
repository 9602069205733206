mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_ttswe.py tests/test_gpu_hooks.py -q -x --durations=15 > $O/pytest_new.log 2>&1; echo "exit $?" >> $O/pytest_new.log
timeout 900 ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/traffic_C4.csv python scripts/traffic.py run C4 4096 5 > $O/traffic_run.log 2>&1
cp gpurun_out/traffic_C4.meta.json $O/ 2>/dev/null
