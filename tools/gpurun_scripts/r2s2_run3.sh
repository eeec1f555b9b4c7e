python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants_bitwise" > gpurun_out/s2_t3.log 2>&1
python tools/option_ab.py aggregate_variant 0 2 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py aggregate_variant 0 2 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
