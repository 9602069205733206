mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
for cr in 256 512; do
  TTSW_CHUNK_ROWS=$cr timeout 600 python scripts/time_step.py C4 4096 12 2> $O/steps_cr$cr.err | cut -c1-150 > $O/steps_cr$cr.txt
  tail -4 $O/steps_cr$cr.txt
done
timeout 600 python scripts/bench_round.py 4097 12288 128 3 > $O/round128.txt 2>&1; tail -2 $O/round128.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_caqr_leaf -s 6 -c 1 -f -o $O/leaf python scripts/bench_round.py 4097 12288 128 3 > $O/ncu_leaf.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_caqr_top -s 6 -c 1 -f -o $O/top python scripts/bench_round.py 4097 12288 128 3 > $O/ncu_top.log 2>&1
ls -la $O
