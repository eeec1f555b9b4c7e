"""Host-side profile of the reference-shaped call restore(y, A, model, tree, config)
(plan cache warm): where the wall time of a single-image call goes."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1710_08124_b200 import RestorationConfig, restore, synthetic

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
case = synthetic.baseline_case(name)
P = synthetic.CONFIGS[name]["patch_dim"] if "patch_dim" in synthetic.CONFIGS[name] else 64
model = synthetic.synthetic_gmm(200, P, 0, 0.95)
tree = synthetic.baseline_tree(model)
cfg = RestorationConfig(sigma=case.sigma8, spacing=case.spacing, seed=0)
for _ in range(3):
    restore(case.y, case.A, model, tree, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 50
for _ in range(n):
    restore(case.y, case.A, model, tree, cfg)
print(f"{name}: {1e3 * (time.perf_counter() - t0) / n:.3f} ms per restore() call")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    restore(case.y, case.A, model, tree, cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
