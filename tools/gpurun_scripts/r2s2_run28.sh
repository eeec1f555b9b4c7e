python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_multiproc.py -m gpu -x -q > gpurun_out/s2_t28.log 2>&1
python bench.py --workload cfg5-strip --no-cpu-baseline --steps 10 > gpurun_out/s2_strip2.json 2>&1
python bench.py --workload cfg5-strip --no-cpu-baseline --steps 10 --option aggregate_variant=0 > gpurun_out/s2_strip0.json 2>&1
