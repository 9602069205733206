export TTSW_PROFILE_TSQR=1
for cfg in "4097 12288 126 3 1e-10 46" "4097 12288 216 3 1e-10 40" "12288 4097 300 3 1e-10 80" "4097 12288 456 3 1e-10 100"; do
  timeout 120 python scripts/bench_round.py $cfg >> gpurun_out/ub_round3.log 2>&1
done
unset TTSW_PROFILE_TSQR
timeout 300 python scripts/time_step.py C4 4096 6 > gpurun_out/c4_v7.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_v7.log 2>&1
