python -m pytest tests/test_gpu_parity.py -m gpu -x -q -W ignore -k "variants or golden or lo_eq_hi or host_pipeline" > gpurun_out/t10.log 2>&1; tail -2 gpurun_out/t10.log
for v in 1 0; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --option aggregate_variant=$v > gpurun_out/b10_a$v.json 2>&1; done
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --option aggregate_variant=1 --precision fp32-state > gpurun_out/b10_a1_fp32.json 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --batch 8 --option aggregate_variant=1 > gpurun_out/b10_b8_a1.json 2>&1
