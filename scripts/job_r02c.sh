mkdir -p gpurun_out/r02c
O=gpurun_out/r02c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
cp -r gpurun_out/long_parity $O/ 2>/dev/null
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
for t in 16 32 64; do
  timeout 900 python bench.py --config C5 --members 64 --member-threads $t --steps 2 --warmup 2 --no-cpu-baseline > $O/bench_C5_t$t.json 2> $O/bench_C5_t$t.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python scripts/time_step.py C4 4096 1 > $O/ncu_launch.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python scripts/time_step.py C3 32 1 > $O/racecheck_C3_N32.log 2>&1; echo "racecheck exit $?" >> $O/racecheck_C3_N32.log
