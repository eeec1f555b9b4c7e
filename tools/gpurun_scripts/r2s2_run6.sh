mkdir -p /tmp/ncu
ncu -f --set full --import-source on --clock-control none -k regex:aggregate_tiles --launch-skip 2 -c 1 -o /tmp/ncu/agg_tiles python tools/prof_run.py 64 1024 tensor 1 aggregate_variant=2 > gpurun_out/s2_ncu_agg.log 2>&1
python tools/ncu_summary.py /tmp/ncu/agg_tiles.ncu-rep > gpurun_out/s2_ncu_agg_tiles.txt 2>&1
cp /tmp/ncu/agg_tiles.ncu-rep gpurun_out/
