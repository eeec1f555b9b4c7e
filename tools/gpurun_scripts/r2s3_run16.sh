timeout 600 python -m pytest tests/test_gpu_fp32_state.py -m gpu -x -q -k "wiener_tc_matches" > gpurun_out/s3_t16.log 2>&1
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 --steps 5 > gpurun_out/s3_wtc3.json 2> gpurun_out/s3_wtc3.err
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=2 --steps 5 > gpurun_out/s3_wtc2.json 2> gpurun_out/s3_wtc2.err
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 --steps 5 --batch 8 > gpurun_out/s3_wtc3_b8.json 2> gpurun_out/s3_wtc3_b8.err
