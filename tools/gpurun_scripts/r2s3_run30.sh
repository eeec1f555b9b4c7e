python -m pytest tests -m gpu -q > gpurun_out/s3_gputests5.log 2>&1
python __graft_entry__.py smoke > gpurun_out/s3_smoke5.log 2>&1
for w in cfg4a cfg4b; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3_lt_$w.json 2>&1; done
python bench.py > gpurun_out/s3_last_default.json 2> gpurun_out/s3_last_default.err
