set -x
python bench.py > gpurun_out/bench.log 2>&1
python bench.py --workload cfg5-strip > gpurun_out/bench_strip.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
for k in "select_level_ws2:4" "wiener_dmma:0" "aggregate_cover:0" "extract_cols:0"; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --import-source on --clock-control none -k regex:$name --launch-skip $skip -c 1 -o gpurun_out/full_$name python tools/prof_run.py 64 1024 tensor > gpurun_out/ncu_$name.log 2>&1
done
