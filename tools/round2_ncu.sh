# full ncu captures of the top kernels; summaries written on the box, the
# reports themselves deleted (gpurun_out must stay under 64 MiB)
mkdir -p /tmp/ncu
for k in "select_level_ws2:4" "wiener_dmma:0" "aggregate_cover:0" "extract_cols:0" "rescore_fp64:3"; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --import-source on --clock-control none -k regex:$name --launch-skip $skip -c 1 -o /tmp/ncu/$name python tools/prof_run.py 64 1024 tensor > gpurun_out/final_ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep > gpurun_out/final_ncu_$name.txt 2>&1
done
ls -la /tmp/ncu > gpurun_out/final_ncu_sizes.txt
cp /tmp/ncu/select_level_ws2.ncu-rep gpurun_out/ 2>/dev/null
