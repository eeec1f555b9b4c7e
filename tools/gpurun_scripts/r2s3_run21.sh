timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants_bitwise and wiener_ws" > gpurun_out/s3_t21.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-opt-in --option wiener_ws=1 > gpurun_out/s3_wws1.json 2> gpurun_out/s3_wws1.err
timeout 300 python bench.py --no-cpu-baseline --no-opt-in > gpurun_out/s3_wws0.json 2> gpurun_out/s3_wws0.err
