# full ncu captures of the top kernels (one launch each, cfg5 64 x 1024^2); summaries on the box
mkdir -p /tmp/ncu
for k in "select_level_ws2:4" "wiener_dmma:0" "aggregate_tiles:0" "extract_cols:0" "verify_kernel:0" "repair_cta_kernel:0"; do
  name=${k%%:*}; skip=${k##*:}
  ncu -f --set full --import-source on --clock-control none -k regex:$name --launch-skip $skip -c 1 -o /tmp/ncu/$name python tools/prof_run.py 64 1024 tensor > gpurun_out/g_ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep > gpurun_out/g_ncu_$name.txt 2>&1
done
cp /tmp/ncu/aggregate_tiles.ncu-rep gpurun_out/ 2>/dev/null
