timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s3_t25.log 2>&1
timeout 600 python tools/level_spans.py 8 1024 > gpurun_out/s3_level_spans_b8b.log 2>&1
timeout 300 python bench.py --batch 8 --no-cpu-baseline --no-opt-in > gpurun_out/s3_b8_split.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-opt-in > gpurun_out/s3_b64_split.json 2>&1
