python -m pytest tests -m gpu -q > gpurun_out/s3_gputests4.log 2>&1
python __graft_entry__.py smoke > gpurun_out/s3_smoke4.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/s3_final20.json 2> gpurun_out/s3_final20.err
for w in cfg1 cfg2 cfg3; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3_final_$w.json 2>&1; done
