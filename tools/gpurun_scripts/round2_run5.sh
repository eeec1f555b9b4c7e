for L in 2 6; do python tools/trace_ws.py $L 64 > gpurun_out/trace5_L$L.log 2>&1; done
