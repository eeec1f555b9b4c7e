timeout 600 python -m pytest tests/test_gpu_fp32_state.py -m gpu -x -q -k "wiener_tc_matches" > gpurun_out/s3_t4.log 2>&1
FEPLL_WTC_STORE=1 timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 > gpurun_out/s3_fp32_tc_bulk.json 2> gpurun_out/s3_fp32_tc_bulk.err
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 > gpurun_out/s3_fp32_tc.json 2> gpurun_out/s3_fp32_tc.err
FEPLL_WTC_STORE=1 timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 --batch 8 > gpurun_out/s3_fp32_tc_bulk_b8.json 2> gpurun_out/s3_fp32_tc_bulk_b8.err
