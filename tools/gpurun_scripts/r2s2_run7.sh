python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants_bitwise or lo_eq_hi" > gpurun_out/s2_t7.log 2>&1
python tools/option_ab.py aggregate_variant 2 0 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py aggregate_variant 2 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
mkdir -p /tmp/ncu
ncu -f --set full --import-source on --clock-control none -k regex:aggregate_tiles --launch-skip 2 -c 1 -o /tmp/ncu/agg_tiles python tools/prof_run.py 64 1024 tensor 1 aggregate_variant=2 > gpurun_out/s2_ncu_agg.log 2>&1
python tools/ncu_summary.py /tmp/ncu/agg_tiles.ncu-rep > gpurun_out/s2_ncu_agg_tiles.txt 2>&1
cp /tmp/ncu/agg_tiles.ncu-rep gpurun_out/
