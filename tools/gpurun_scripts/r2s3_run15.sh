python -m pytest tests -m gpu -q > gpurun_out/s3_gputests2.log 2>&1
python __graft_entry__.py smoke > gpurun_out/s3_smoke2.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/s3_default20.json 2> gpurun_out/s3_default20.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3_reference.json 2>&1
