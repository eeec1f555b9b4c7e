python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q > gpurun_out/s2_t18.log 2>&1
python tools/option_ab.py pdl 1 0 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py pdl 1 0 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
python tools/level_spans.py 8 > gpurun_out/s2_spans8.txt 2>&1
python bench.py --batch 8 --no-cpu-baseline > gpurun_out/s2_bench8.json 2>&1
