ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launch8.csv python tools/prof_run.py 8 1024 tensor 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launch64.csv python tools/prof_run.py 64 1024 tensor 1 > /dev/null 2>&1
