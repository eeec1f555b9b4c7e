timeout 600 python tools/restore_profile.py cfg1 > gpurun_out/s3_restore_profile_cfg1c.log 2>&1
timeout 900 python -m pytest tests/test_solver_scenarios.py tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q > gpurun_out/s3_t13.log 2>&1
for w in cfg1 cfg2 cfg3 cfg4a cfg4b; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3_$w.json 2>&1; done
python - <<'PY' > gpurun_out/s3_times_check.log 2>&1
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1710_08124_b200 import RestorationConfig, restore, synthetic
case = synthetic.baseline_case("cfg2")
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
cfg = RestorationConfig(sigma=case.sigma8, spacing=case.spacing, seed=0)
for k in range(3):
    x, st = restore(case.y, case.A, model, tree, cfg)
    print([{a: round(b * 1e6, 1) for a, b in it.times.items()} for it in st.iterations][:2], st.init_seconds, st.total_seconds)
PY
