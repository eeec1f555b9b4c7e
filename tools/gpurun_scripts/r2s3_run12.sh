timeout 600 python tools/restore_profile.py cfg1 > gpurun_out/s3_restore_profile_cfg1b.log 2>&1
timeout 900 python -m pytest tests/test_solver_scenarios.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s3_t12.log 2>&1
for w in cfg1 cfg2 cfg3 cfg4a cfg4b; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3_$w.json 2>&1; done
