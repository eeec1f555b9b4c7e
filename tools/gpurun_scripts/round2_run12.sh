python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -m gpu -x -q -W ignore -k "ties or variants or golden or select_kernel" > gpurun_out/t12.log 2>&1; tail -3 gpurun_out/t12.log
for o in 1 0; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --option local_rescore=$o > gpurun_out/b12_l$o.json 2>&1; done
for o in 1 0; do python bench.py --steps 10 --warmup 3 --batch 8 --no-cpu-baseline --option local_rescore=$o > gpurun_out/b12_b8_l$o.json 2>&1; done
for o in 1 0; do python bench.py --workload cfg1 --steps 10 --warmup 3 --no-cpu-baseline --option local_rescore=$o > gpurun_out/b12_cfg1_l$o.json 2>&1; done
