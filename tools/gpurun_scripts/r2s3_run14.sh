for v in 0 1 2 3; do
FEPLL_EXTRACT_VARIANT=$v timeout 300 python bench.py --precision fp32-state --option wiener_tc=1 --no-cpu-baseline --steps 5 > gpurun_out/s3_ext_v${v}_fp32.json 2>&1
FEPLL_EXTRACT_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/s3_ext_v${v}_fp64.json 2>&1
done
