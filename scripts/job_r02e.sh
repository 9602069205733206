mkdir -p gpurun_out/r02e
O=gpurun_out/r02e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 3000 python -m pytest tests -q -m gpu --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/ 2>/dev/null
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python scripts/time_step.py C4 4096 6 > $O/ncu_launch.log 2>&1
tail -5 $O/pytest_gpu.log; cat $O/bench_C4.json; tail -2 $O/smoke.log
