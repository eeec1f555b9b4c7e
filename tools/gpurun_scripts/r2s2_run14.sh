python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q > gpurun_out/s2_t14.log 2>&1
python tools/option_ab.py rescore_group 1 0 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py rescore_group 1 0 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
