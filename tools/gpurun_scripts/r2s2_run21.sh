python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q > gpurun_out/s2_t21.log 2>&1
python tools/level_spans.py 64 > gpurun_out/s2_spans64.txt 2>&1
python tools/option_ab.py pdl 1 > gpurun_out/s2_ab64.txt 2>&1
