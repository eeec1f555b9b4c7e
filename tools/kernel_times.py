"""Per-kernel device time of one 64 x 1024^2 restore (torch profiler / CUPTI),
grouped by kernel name, plus the tree-level kernels per level."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ys = np.stack([synthetic.baseline_case("cfg5", 1024, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
y = torch.from_numpy(ys).cuda()
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
r.run(y); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.run(y); torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
tot = collections.Counter(); cnt = collections.Counter()
for e in ev:
    tot[e.name[:90]] += e.device_time; cnt[e.name[:90]] += 1
allt = sum(tot.values())
print(f"total kernel time {allt/1000:.3f} ms")
for k, v in tot.most_common(25):
    print(f"{v/1000:8.3f} ms {cnt[k]:4d}x  {k}")
lv = [e.device_time for e in ev if "select_level" in e.name]
if len(lv) % 7 == 0:
    print("per-level us:", np.round(np.array(lv).reshape(-1, 7).mean(axis=0)).astype(int).tolist())
