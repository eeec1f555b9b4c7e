python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_solver_scenarios.py -m gpu -x -q > gpurun_out/s2_t29.log 2>&1
for w in cfg4a cfg4b; do
python bench.py --workload $w --no-cpu-baseline > gpurun_out/s2_${w}_d1.json 2>&1
python bench.py --workload $w --no-cpu-baseline --option defer=0 > gpurun_out/s2_${w}_d0.json 2>&1
done
