timeout 300 python scripts/sweeps_tmp.py
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 80 --csv --log-file gpurun_out/launch_v2e.csv python scripts/time_step.py C2 1024 3 > /dev/null 2>&1
