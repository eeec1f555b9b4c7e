python -m pytest tests -m gpu -q > gpurun_out/s3_gputests3.log 2>&1
python __graft_entry__.py smoke > gpurun_out/s3_smoke3.log 2>&1
python bench.py > gpurun_out/s3_final_default.json 2> gpurun_out/s3_final_default.err
python bench.py --workload cfg5-strip --no-cpu-baseline > gpurun_out/s3_final_strip.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-opt-in > gpurun_out/s3_ncu_launch_default.log 2>&1
