python -m pytest tests -m gpu -x -q > gpurun_out/s2_t22.log 2>&1
python tools/option_ab.py defer 1 0 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py defer 1 0 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
