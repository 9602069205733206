mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
timeout 3000 python -m pytest tests -q -m gpu --durations=8 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/ 2>/dev/null
tail -16 $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
cat $O/bench_C4.json
timeout 600 python bench.py --config C3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
cat $O/bench_C3.json
