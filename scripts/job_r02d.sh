mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/ 2>/dev/null
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --rep dense > $O/bench_C4_dense.json 2> $O/bench_C4_dense.err
timeout 600 python bench.py --config C3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 600 python bench.py --config C1 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err
/usr/bin/time -v timeout 1750 python bench.py --impl reference > $O/bench_ref_C4.json 2> $O/bench_ref_C4.err
