mkdir -p gpurun_out/r02g
O=gpurun_out/r02g
TTSW_SKETCH_VERBOSE=1 timeout 1200 python -m pytest tests/test_gpu_sketch.py -x -q > $O/pytest_sketch.log 2>&1; echo "pytest exit $?" >> $O/pytest_sketch.log
tail -40 $O/pytest_sketch.log
timeout 600 python scripts/time_step.py C4 4096 10 > $O/steps.txt 2> $O/steps.err
cut -c1-200 $O/steps.txt
