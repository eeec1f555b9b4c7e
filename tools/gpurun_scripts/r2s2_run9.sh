python -m pytest tests -m gpu -q > gpurun_out/s2_gputests.log 2>&1
mkdir -p /tmp/ncu
ncu -f --set full --import-source on --clock-control none -k regex:wiener_dmma --launch-skip 1 -c 1 -o /tmp/ncu/wiener python tools/prof_run.py 64 1024 tensor 1 > gpurun_out/s2_ncu_w.log 2>&1
python tools/ncu_summary.py /tmp/ncu/wiener.ncu-rep > gpurun_out/s2_ncu_wiener.txt 2>&1
cp /tmp/ncu/wiener.ncu-rep gpurun_out/
