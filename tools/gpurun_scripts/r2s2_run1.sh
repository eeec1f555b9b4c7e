# session-2 check: GPU suite, default bench, FP64 pipe-mix microbenchmark
./tools/fp64_mix_bench > gpurun_out/s2_fp64mix.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/s2_gputests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
