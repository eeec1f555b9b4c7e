mkdir -p /tmp/ncu
ncu -f --set full --import-source on --cache-control none --clock-control none -k regex:rescore_group --launch-skip 10 -c 1 -o /tmp/ncu/rg8 python tools/prof_run.py 8 1024 tensor 1 > gpurun_out/s2_ncu_rg.log 2>&1
ncu -f --set full --import-source on --cache-control none --clock-control none -k regex:rescore_fp64 --launch-skip 10 -c 1 -o /tmp/ncu/rf8 python tools/prof_run.py 8 1024 tensor 1 rescore_group=0 > gpurun_out/s2_ncu_rf.log 2>&1
cp /tmp/ncu/rg8.ncu-rep /tmp/ncu/rf8.ncu-rep gpurun_out/
