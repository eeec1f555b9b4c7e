python -m pytest tests -m gpu -x -q -W ignore > gpurun_out/t13.log 2>&1; tail -3 gpurun_out/t13.log
python __graft_entry__.py smoke > gpurun_out/smoke13.log 2>&1; tail -2 gpurun_out/smoke13.log
bash tools/round2_ncu.sh
