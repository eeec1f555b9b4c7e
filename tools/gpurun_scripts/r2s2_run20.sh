python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_fp32_state.py -m gpu -x -q > gpurun_out/s2_t20.log 2>&1
python tools/option_ab.py wiener_split 1 0 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py wiener_split 1 0 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
python tools/option_ab.py wiener_split 1 0 --precision fp32-state > gpurun_out/s2_ab64f.txt 2>&1
