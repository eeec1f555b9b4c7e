timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_solver_scenarios.py -m gpu -x -q > gpurun_out/s3_t29.log 2>&1
timeout 600 python tools/level_spans.py 8 1024 > gpurun_out/s3_level_spans_b8c.log 2>&1
for w in cfg1 cfg2 cfg3; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3_lt_$w.json 2>&1; done
timeout 300 python bench.py --batch 8 --no-cpu-baseline --no-opt-in > gpurun_out/s3_lt_b8.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-opt-in > gpurun_out/s3_lt_b64.json 2>&1
