"""Small driver for ncu / compute-sanitizer: one (or reps) restore of a
BASELINE config at a chosen size through the public restore_batch API.
python tools/cfg_run.py <cfg> <size> <batch> <mode> [reps] [use_tree]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
cfg = sys.argv[1]
size = int(sys.argv[2])
B = int(sys.argv[3])
mode = sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
use_tree = bool(int(sys.argv[6])) if len(sys.argv) > 6 else True
cases = [synthetic.baseline_case(cfg, size, image_seed=i, noise_seed=1000 + i) for i in range(B)]
A = cases[0].A
spec = synthetic.CONFIGS[cfg]
model = synthetic.synthetic_gmm(200 if use_tree else 40, spec["patch_dim"], 0, 0.95)
tree = synthetic.baseline_tree(model) if use_tree else None
r = Restorer(A, model, tree, RestorationConfig(sigma=spec["sigma"], spacing=spec["spacing"], seed=0,
                                               use_tree=use_tree), batch=B, mode=mode)
y = torch.from_numpy(np.stack([c.y for c in cases])).cuda()
for _ in range(reps):
    r.run(y)
torch.cuda.synchronize()
r.check_status()
print("ok", cfg, size, B, mode, r.counters()[0])
