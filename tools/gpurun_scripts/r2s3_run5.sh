timeout 900 python tools/wtc_diag.py 64 1024 > gpurun_out/s3_wtc_diag64.log 2>&1
