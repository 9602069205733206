mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_ubench scripts/ubench/fp64_ubench.cu && /tmp/fp64_ubench > $O/ubench.txt 2>&1
timeout 900 python scripts/diag_numrank.py 4096 8 > $O/numrank.txt 2>&1
TTSW_PROFILE_TSQR=1 TTSW_PROFILE_RHS=1 timeout 900 python scripts/time_step.py C4 4096 10 > $O/steps.txt 2> $O/steps_prof.txt
tail -30 $O/numrank.txt; cat $O/ubench.txt
