timeout 600 python tools/wtc_prof.py 64 > gpurun_out/s3_wtc_prof.log 2>&1
