mkdir -p gpurun_out/r02p
O=gpurun_out/r02p
timeout 1500 python bench.py --config C5 --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_C5_t16.json 2> $O/bench_C5_t16.err; cat $O/bench_C5_t16.json | cut -c1-400
timeout 1500 python bench.py --config C5 --no-cpu-baseline --steps 3 --warmup 3 --member-threads 8 > $O/bench_C5_t8.json 2> $O/bench_C5_t8.err; cat $O/bench_C5_t8.json | cut -c1-400
timeout 600 python bench.py --config C2 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err; cut -c1-300 $O/bench_C2.json
timeout 600 python bench.py --config C1 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err; cut -c1-300 $O/bench_C1.json
