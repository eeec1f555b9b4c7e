"""Per-level durations of the tree-level kernel (one restore, CUPTI)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
ys = torch.from_numpy(np.stack([c.y] * B)).cuda()
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
r.run(ys); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.run(ys); torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "select_level" in e.name],
            key=lambda e: e.time_range.start)
t = np.array([e.device_time for e in ev]).reshape(-1, 7)
print("per-level us (mean over iterations):", np.round(t.mean(axis=0)).astype(int).tolist(), "sum", int(t.sum()))
