mkdir -p gpurun_out/r02l
O=gpurun_out/r02l
timeout 1500 ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic_C4.csv python scripts/traffic.py run C4 4096 8 > $O/traffic.log 2>&1
cp gpurun_out/traffic_C4.csv gpurun_out/traffic_C4.meta.json $O/
tail -3 $O/traffic.log
