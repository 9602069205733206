mkdir -p gpurun_out/r02z4
O=gpurun_out/r02z4
timeout 1500 python bench.py --config C5 --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_C5_t8.json 2> $O/bench_C5_t8.err; cut -c1-260 $O/bench_C5_t8.json
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_jacobi_cluster -s 2 -c 2 -f -o $O/k_jacobi_cluster python scripts/traffic.py run C4 4096 20 > $O/ncu_jacobi.log 2>&1; tail -2 $O/ncu_jacobi.log
ls -la $O
