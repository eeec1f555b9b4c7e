python -m pytest tests/test_gpu_fp32_state.py -m gpu -q > gpurun_out/s3_t27.log 2>&1
