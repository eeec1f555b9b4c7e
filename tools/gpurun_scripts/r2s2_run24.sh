python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_solver_scenarios.py -m gpu -x -q > gpurun_out/s2_t24.log 2>&1
python tools/option_ab.py defer 1 0 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py defer 1 0 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"verify|repair" --log-file gpurun_out/s2_vr64.csv python tools/prof_run.py 64 1024 tensor 1 > /dev/null 2>&1
