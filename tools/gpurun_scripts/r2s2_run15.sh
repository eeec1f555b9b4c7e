ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:rescore --log-file gpurun_out/s2_rs1.csv python tools/prof_run.py 64 1024 tensor 1 rescore_group=1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:rescore --log-file gpurun_out/s2_rs0.csv python tools/prof_run.py 64 1024 tensor 1 rescore_group=0 > /dev/null 2>&1
