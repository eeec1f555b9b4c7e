# level spans (imbalance check) + ncu full capture of the tcgen05 Wiener kernel + launch list in fp32-state/wiener_tc mode
timeout 600 python tools/level_spans.py 64 1024 > gpurun_out/s3_level_spans.log 2>&1
mkdir -p /tmp/ncu
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:wiener_tc --launch-skip 1 -c 1 -o /tmp/ncu/wiener_tc python tools/prof_run.py 64 1024 tensor 1 wiener_tc=1 fp32-state > gpurun_out/s3_ncu_wiener_tc.log 2>&1
python tools/ncu_summary.py /tmp/ncu/wiener_tc.ncu-rep > gpurun_out/s3_ncu_wiener_tc.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches_fp32tc.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --precision fp32-state --option wiener_tc=1 > gpurun_out/s3_ncu_launch.log 2>&1
