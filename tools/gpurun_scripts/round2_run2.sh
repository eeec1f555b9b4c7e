set -x
python -m pytest tests/test_solver_scenarios.py tests/test_gpu_parity.py -m gpu -x -q -W ignore -k "scenario or reference_runs or properties or exact_profile or surrogate or optimality or worker or profile or tree_profile or variants or host_pipeline or golden" > gpurun_out/t2.log 2>&1; tail -3 gpurun_out/t2.log
for w in cfg5-batch; do python bench.py --steps 10 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; tail -c 600 gpurun_out/b_$w.json; done
python bench.py --steps 10 --warmup 3 --graph 0 --no-cpu-baseline > gpurun_out/b_nograph.json 2>&1; tail -c 300 gpurun_out/b_nograph.json
python bench.py --steps 10 --warmup 3 --batch 8 --no-cpu-baseline > gpurun_out/b_batch8.json 2>&1
python bench.py --steps 10 --warmup 3 --batch 8 --graph 0 --no-cpu-baseline > gpurun_out/b_batch8_nograph.json 2>&1
for w in cfg1 cfg2 cfg3 cfg4a cfg4b; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; tail -c 300 gpurun_out/b_$w.json; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.json 2>&1
