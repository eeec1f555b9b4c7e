python -m pytest tests -m gpu -x -q > gpurun_out/s2_gputests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
python bench.py --batch 8 --no-cpu-baseline > gpurun_out/s2_bench8.json 2>&1
