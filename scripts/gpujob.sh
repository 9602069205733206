set -x
timeout 1500 python -m pytest tests -q -m gpu --durations=8 > gpurun_out/pytest_gpu_r01b.log 2>&1; tail -14 gpurun_out/pytest_gpu_r01b.log
timeout 600 python bench.py --steps 50 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json; tail -3 gpurun_out/bench_r01b.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_r01b.json 2>&1; cat gpurun_out/bench_ref_r01b.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
