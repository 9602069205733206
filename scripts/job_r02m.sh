mkdir -p gpurun_out/r02m
O=gpurun_out/r02m
timeout 1200 python -m pytest tests/test_gpu_sketch.py tests/test_gpu_parity.py -x -q -k "sketch or round_ or caqr" > $O/pytest_a.log 2>&1; tail -5 $O/pytest_a.log
TTSW_SKETCH_VERBOSE=1 TTSW_PROFILE_TSQR=1 TTSW_PROFILE_RHS=1 timeout 900 python scripts/time_step.py C4 4096 25 > $O/steps.txt 2> $O/steps_prof.txt
cut -c1-150 $O/steps.txt
