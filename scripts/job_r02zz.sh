mkdir -p gpurun_out/r02z3
O=gpurun_out/r02z3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 3300 python -m pytest tests -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -18 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; cat $O/bench_C4.json
timeout 600 python bench.py --config C3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err; cut -c1-200 $O/bench_C3.json
TTSW_PROFILE_SYNC=1 timeout 600 python scripts/time_step.py C4 4096 8 > $O/steps_sync.txt 2> $O/steps_sync.err; grep "step wall" $O/steps_sync.err | tail -3
