for o in 0 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --option l2_prefetch=$o > gpurun_out/b4_pf$o.json 2>&1; done
