python tools/option_ab.py wiener_rw 8 16 > gpurun_out/s2_ab64.txt 2>&1
python tools/option_ab.py wiener_rw 8 16 --batch 8 > gpurun_out/s2_ab8.txt 2>&1
