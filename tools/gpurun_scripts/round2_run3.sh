python -m pytest tests/test_tree_build.py tests/test_gpu_parity.py -m gpu -x -q -W ignore -k "tree or variants" > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3_pf1.json 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --option l2_prefetch=0 > gpurun_out/b3_pf0.json 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3_pf1b.json 2>&1
