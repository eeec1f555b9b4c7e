# full ncu captures of the top kernels (one launch each, cfg5 64 x 1024^2, FP64 default); summaries on the box
mkdir -p /tmp/ncu
for k in "select_level_ws2:4" "wiener_ws:0" "aggregate_tiles:0" "extract_cols:0" "verify_kernel:0"; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:$name --launch-skip $skip -c 1 -o /tmp/ncu/$name python tools/prof_run.py 64 1024 tensor > gpurun_out/s3_ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep > gpurun_out/s3_ncu_$name.txt 2>&1
done
