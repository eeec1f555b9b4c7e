python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_solver_scenarios.py tests/test_tree_build.py -m gpu -x -q -W ignore > gpurun_out/t7.log 2>&1; tail -3 gpurun_out/t7.log
for o in 1 0; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --option rescore_by_node=$o > gpurun_out/b7_r$o.json 2>&1; done
for o in 1 0; do python bench.py --steps 10 --warmup 3 --batch 8 --no-cpu-baseline --option rescore_by_node=$o > gpurun_out/b7_b8_r$o.json 2>&1; done
for w in cfg1 cfg4a; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b7_$w.json 2>&1; done
