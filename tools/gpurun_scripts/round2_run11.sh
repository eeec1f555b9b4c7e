python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32_state.py -m gpu -x -q -W ignore -k "golden or full_size or operator or adjoint or cfg2" > gpurun_out/t11.log 2>&1; tail -3 gpurun_out/t11.log
for w in cfg3 cfg4a cfg4b; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b11_$w.json 2>&1; done
