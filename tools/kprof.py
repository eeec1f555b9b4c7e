"""Per-kernel device time of one restore (torch.profiler / CUPTI, warm caches)."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
ys = torch.from_numpy(np.stack([c.y] * B)).cuda()
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
r.run(ys); r.run(ys); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.run(ys); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
for e in evs:
    a = agg[e.name[:70]]; a[0] += 1; a[1] += e.device_time
tot = sum(a[1] for a in agg.values())
print(f"B={B} total kernel us {tot:.0f}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"  {k:70s} {n:4d} {t:9.0f} us avg {t / n:8.1f}")
# timeline span
t0 = min(e.time_range.start for e in evs); t1 = max(e.time_range.end for e in evs)
print("span us", t1 - t0)
