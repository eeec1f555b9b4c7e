python -m pytest tests -m gpu -q > gpurun_out/s3_gputests6.log 2>&1
python __graft_entry__.py smoke > gpurun_out/s3_smoke6.log 2>&1
for w in cfg1 cfg2 cfg3; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3_nt_$w.json 2>&1; done
timeout 300 python bench.py --batch 8 --no-cpu-baseline --no-opt-in > gpurun_out/s3_nt_b8.json 2>&1
python bench.py > gpurun_out/s3_nt_default.json 2> gpurun_out/s3_nt_default.err
