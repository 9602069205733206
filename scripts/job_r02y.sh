mkdir -p gpurun_out/r02y
O=gpurun_out/r02y
for mr in 160 128 112; do
  TTSW_SKETCH_MIN_R=$mr timeout 600 python scripts/time_step.py C4 4096 14 2> $O/steps_mr$mr.err | cut -c1-150 > $O/steps_mr$mr.txt
  echo "min_r $mr"; tail -6 $O/steps_mr$mr.txt | awk '{print $1,$2,$3}'
done
