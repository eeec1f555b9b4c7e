# compute-sanitizer on the mbarrier / tcgen05 pipelines (small restores)
for t in racecheck synccheck memcheck; do
  compute-sanitizer --tool $t --error-exitcode 9 python tools/cfg_run.py cfg1 96 2 tensor > gpurun_out/san_${t}_cfg1.log 2>&1; echo "$t cfg1 rc=$?" >> gpurun_out/san_summary.txt
done
compute-sanitizer --tool racecheck --error-exitcode 9 python tools/cfg_run.py cfg4a 96 1 tensor > gpurun_out/san_racecheck_cfg4a.log 2>&1; echo "racecheck cfg4a rc=$?" >> gpurun_out/san_summary.txt
compute-sanitizer --tool memcheck --error-exitcode 9 python tools/cfg_run.py cfg4b 96 1 tensor > gpurun_out/san_memcheck_cfg4b.log 2>&1; echo "memcheck cfg4b rc=$?" >> gpurun_out/san_summary.txt
compute-sanitizer --tool racecheck --error-exitcode 9 python tools/cfg_run.py cfg1 64 1 tensor 1 0 > gpurun_out/san_racecheck_notree.log 2>&1; echo "racecheck notree rc=$?" >> gpurun_out/san_summary.txt
# launch lists of the small configs (kernel durations, cold cache, serialised)
for c in cfg1 cfg4b; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/cfg_run.py $c 512 1 tensor 1 > gpurun_out/ncu_l_$c.log 2>&1
done
# full captures: select_tc (P=100), FFT solve (cfg3), CG (cfg4b)
ncu --set full --import-source on --clock-control none -k regex:select_level_tc --launch-skip 3 -c 1 -o gpurun_out/full_select_tc python tools/cfg_run.py cfg4a 512 1 tensor > gpurun_out/ncu_tc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fft_cols_filter --launch-skip 2 -c 1 -o gpurun_out/full_fft python tools/cfg_run.py cfg3 512 1 tensor > gpurun_out/ncu_fft.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:cg_kernel --launch-skip 1 -c 1 -o gpurun_out/full_cg python tools/cfg_run.py cfg4b 510 1 tensor > gpurun_out/ncu_cg.log 2>&1
