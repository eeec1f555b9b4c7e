timeout 600 python -m pytest tests/test_gpu_fp32_state.py -m gpu -x -q -k "wiener_tc_matches" > gpurun_out/s3_t18.log 2>&1
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 > gpurun_out/s3_wtc_alt.json 2> gpurun_out/s3_wtc_alt.err
