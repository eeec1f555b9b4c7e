timeout 600 python tools/level_spans.py 8 1024 > gpurun_out/s3_level_spans_b8.log 2>&1
