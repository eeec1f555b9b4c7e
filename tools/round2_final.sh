# round-2 evidence: bench lines for every workload, the reference arm, the
# ncu launch list of the default bench
python bench.py > gpurun_out/final_cfg5-batch.json 2> gpurun_out/final_cfg5-batch.err
python bench.py --workload cfg5-strip > gpurun_out/final_cfg5-strip.json 2>&1
for w in cfg1 cfg2 cfg3 cfg4a cfg4b; do python bench.py --workload $w > gpurun_out/final_$w.json 2>&1; done
python bench.py --precision fp32-state --no-cpu-baseline > gpurun_out/final_cfg5-batch-fp32.json 2>&1
python bench.py --batch 8 --no-cpu-baseline > gpurun_out/final_cfg5-batch8.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_reference.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1
