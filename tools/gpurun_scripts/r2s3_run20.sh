( time python bench.py > gpurun_out/s3_default_optin.json 2> gpurun_out/s3_default_optin.err ) 2> gpurun_out/s3_default_optin.time
python bench.py --batch 8 --no-cpu-baseline > gpurun_out/s3_b8_optin.json 2>&1
