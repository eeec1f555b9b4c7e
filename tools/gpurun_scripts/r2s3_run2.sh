timeout 600 python tools/wtc_diag.py 4 1024 > gpurun_out/s3_wtc_diag.log 2>&1
