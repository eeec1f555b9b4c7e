# session-2 evidence: GPU suite, bench lines for every workload, reference arm, ncu launch list
python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1
python __graft_entry__.py smoke > gpurun_out/f_smoke.log 2>&1
python bench.py > gpurun_out/f_cfg5-batch.json 2> gpurun_out/f_cfg5-batch.err
python bench.py --batch 8 --no-cpu-baseline > gpurun_out/f_cfg5-batch8.json 2>&1
python bench.py --precision fp32-state --no-cpu-baseline > gpurun_out/f_cfg5-batch-fp32.json 2>&1
python bench.py --workload cfg5-strip > gpurun_out/f_cfg5-strip.json 2>&1
for w in cfg1 cfg2 cfg3 cfg4a cfg4b; do python bench.py --workload $w > gpurun_out/f_$w.json 2>&1; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_reference.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1
