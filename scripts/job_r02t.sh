mkdir -p gpurun_out/r02t
O=gpurun_out/r02t
timeout 1750 python bench.py --impl reference > $O/bench_ref_C4.json 2> $O/bench_ref_C4.err
cat $O/bench_ref_C4.json | cut -c1-900
