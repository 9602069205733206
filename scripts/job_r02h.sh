mkdir -p gpurun_out/r02h
O=gpurun_out/r02h
TTSW_SKETCH_VERBOSE=1 TTSW_PROFILE_TSQR=1 TTSW_PROFILE_RHS=1 timeout 900 python scripts/time_step.py C4 4096 10 > $O/steps.txt 2> $O/steps_prof.txt
timeout 3000 python -m pytest tests -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
rm -rf $O/long_parity; cp -r gpurun_out/long_parity $O/ 2>/dev/null
tail -30 $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
cat $O/bench_C4.json
