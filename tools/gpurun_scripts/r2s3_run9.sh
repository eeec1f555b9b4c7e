# session 3: full GPU suite + smoke + bench lines with the tcgen05 Wiener option
python -m pytest tests -m gpu -q > gpurun_out/s3_gputests.log 2>&1
python __graft_entry__.py smoke > gpurun_out/s3_smoke.log 2>&1
python bench.py > gpurun_out/s3_cfg5-batch.json 2> gpurun_out/s3_cfg5-batch.err
python bench.py --precision fp32-state --option wiener_tc=1 --no-cpu-baseline > gpurun_out/s3_cfg5-batch-fp32tc.json 2>&1
python bench.py --precision fp32-state --no-cpu-baseline > gpurun_out/s3_cfg5-batch-fp32.json 2>&1
python bench.py --precision fp32-state --option wiener_tc=1 --no-cpu-baseline --batch 8 > gpurun_out/s3_cfg5-batch8-fp32tc.json 2>&1
python bench.py --no-cpu-baseline --batch 8 > gpurun_out/s3_cfg5-batch8.json 2>&1
python bench.py --workload cfg5-strip --precision fp32-state --option wiener_tc=1 --no-cpu-baseline > gpurun_out/s3_cfg5-strip-fp32tc.json 2>&1
