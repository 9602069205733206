mkdir -p gpurun_out/r02q
O=gpurun_out/r02q
timeout 1200 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_parity.py -x -q -k "sketch or round_ or caqr" > $O/pytest_a.log 2>&1; tail -3 $O/pytest_a.log
timeout 600 python scripts/time_step.py C4 4096 14 2> $O/steps.err | cut -c1-150 > $O/steps.txt; tail -6 $O/steps.txt
timeout 1500 python bench.py --config C5 --no-cpu-baseline --steps 3 --warmup 3 --member-threads 4 > $O/bench_C5_t4.json 2> $O/bench_C5_t4.err; cat $O/bench_C5_t4.json | cut -c1-300
