python tools/level_spans.py 64 > gpurun_out/s2_spans64.txt 2>&1
python tools/level_spans.py 8 > gpurun_out/s2_spans8.txt 2>&1
