python -m pytest tests/test_gpu_fp32_state.py tests/test_gpu_headline.py tests/test_gpu_parity.py -m gpu -x -q -W ignore > gpurun_out/t9.log 2>&1; tail -3 gpurun_out/t9.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b9_fp64.json 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --precision fp32-state > gpurun_out/b9_fp32.json 2>&1
python bench.py --steps 10 --warmup 3 --batch 8 --no-cpu-baseline --precision fp32-state > gpurun_out/b9_b8_fp32.json 2>&1
