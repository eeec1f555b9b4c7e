python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32_state.py -m gpu -x -q > gpurun_out/s2_t11.log 2>&1
python tools/option_ab.py aggregate_variant 2 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py aggregate_variant 2 --precision fp32-state > gpurun_out/s2_ab64f.txt 2>&1
