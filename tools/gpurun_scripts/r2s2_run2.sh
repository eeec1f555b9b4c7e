./tools/fp64_mix_bench > gpurun_out/s2_fp64mix2.txt 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants_bitwise or cover or aggregate" > gpurun_out/s2_t2.log 2>&1
python tools/option_ab.py aggregate_variant 0 2 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py aggregate_variant 0 2 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
python tools/option_ab.py aggregate_variant 0 2 --precision fp32-state > gpurun_out/s2_ab64f.txt 2>&1
