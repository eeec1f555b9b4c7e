timeout 600 python tools/option_ab.py wiener_ws 0 1 0 1 --batch 64 --reps 5 > gpurun_out/s3_ab_wws64.log 2>&1
timeout 600 python tools/option_ab.py wiener_ws 0 1 0 1 --batch 8 --reps 5 > gpurun_out/s3_ab_wws8.log 2>&1
timeout 600 python tools/option_ab.py wiener_ws 0 1 --batch 1 --size 512 --reps 5 > gpurun_out/s3_ab_wws1.log 2>&1
mkdir -p /tmp/ncu
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:wiener_ws --launch-skip 1 -c 1 -o /tmp/ncu/wiener_ws python tools/prof_run.py 64 1024 tensor 1 wiener_ws=1 > gpurun_out/s3_ncu_wiener_ws.log 2>&1
python tools/ncu_summary.py /tmp/ncu/wiener_ws.ncu-rep > gpurun_out/s3_ncu_wiener_ws.txt 2>&1
