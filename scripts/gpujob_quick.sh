V=33
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_v33.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_v33.log
timeout 900 python bench.py > gpurun_out/bench_C4_v33.json 2> gpurun_out/bench_C4_v33.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_C4_v33.json 2> gpurun_out/bench_ref_C4_v33.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v33.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_v33.log
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2_v33.json 2> gpurun_out/bench_C2_v33.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_v33.csv python scripts/time_step.py C4 4096 1 > gpurun_out/ncu_launch_v33.log 2>&1
tail -3 gpurun_out/pytest_v33.log; cat gpurun_out/bench_C4_v33.json gpurun_out/bench_ref_C4_v33.json; tail -2 gpurun_out/smoke_v33.log
