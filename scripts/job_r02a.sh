mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
timeout 1500 python scripts/long_curve.py C4 4096 500 $O/curve_C4.json > $O/curve_C4.log 2>&1
M=sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for k in k_caqr_update_mma3 k_caqr_leaf; do
  timeout 600 ncu --clock-control none --metrics $M -k regex:$k -s 20 -c 3 --csv --log-file $O/dmma_$k.csv python scripts/time_step.py C4 4096 1 > $O/ncu_$k.log 2>&1
done
