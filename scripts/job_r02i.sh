mkdir -p gpurun_out/r02i
O=gpurun_out/r02i
TTSW_SKETCH_VERBOSE=1 TTSW_PROFILE_TSQR=1 TTSW_PROFILE_RHS=1 timeout 900 python scripts/time_step.py C4 4096 25 > $O/steps.txt 2> $O/steps_prof.txt
cut -c1-220 $O/steps.txt
