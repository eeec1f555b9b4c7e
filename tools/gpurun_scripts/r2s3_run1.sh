# session 3, run 1: tcgen05 Wiener (wiener_tc) first parity + speed
timeout 600 python -m pytest tests/test_gpu_fp32_state.py -m gpu -x -q -k "wiener_tc_matches" > gpurun_out/s3_t1.log 2>&1
echo "rc=$?" >> gpurun_out/s3_t1.log
timeout 900 python -m pytest tests/test_gpu_fp32_state.py -m gpu -q > gpurun_out/s3_t1b.log 2>&1
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline > gpurun_out/s3_fp32_dmma.json 2> gpurun_out/s3_fp32_dmma.err
timeout 300 python bench.py --precision fp32-state --no-cpu-baseline --option wiener_tc=1 > gpurun_out/s3_fp32_tc.json 2> gpurun_out/s3_fp32_tc.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s3_fp64.json 2> gpurun_out/s3_fp64.err
