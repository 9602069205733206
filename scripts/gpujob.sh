V=${V:-33}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_v${V}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_v${V}.log
timeout 900 python bench.py > gpurun_out/bench_C4_v${V}.json 2> gpurun_out/bench_C4_v${V}.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_C4_v${V}.json 2> gpurun_out/bench_ref_C4_v${V}.err
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3_v${V}.json 2> gpurun_out/bench_C3_v${V}.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2_v${V}.json 2> gpurun_out/bench_C2_v${V}.err
timeout 1200 python bench.py --config C5 --members 32 --no-cpu-baseline > gpurun_out/bench_C5_v${V}.json 2> gpurun_out/bench_C5_v${V}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_v${V}.csv python scripts/time_step.py C4 4096 1 > gpurun_out/ncu_launch_v${V}.log 2>&1
timeout 600 python scripts/timeline.py C4 4096 3 1 > gpurun_out/timeline_v${V}.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v${V}.log 2>&1
for k in k_caqr_leaf k_caqr_top k_qrcp_cluster k_svd_qrcp_batch k_maxvol_loop k_fullpiv_cluster; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 25 -c 1 -o gpurun_out/v${V}_$k -f python scripts/time_step.py C4 4096 1 > gpurun_out/ncu_v${V}_$k.log 2>&1
done
