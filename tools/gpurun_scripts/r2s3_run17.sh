timeout 300 ./tools/mma_bench > gpurun_out/s3_mma_bench.txt 2>&1
