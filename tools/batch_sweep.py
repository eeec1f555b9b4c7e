"""Per-image phase cost vs batch size (L2-residency probe): a 1024^2 image's
patch rows are 16 MB (FP32) / 32 MB (FP64), so small batches keep the
gathered rows L2-resident between tree levels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic

c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
for B in [int(b) for b in (sys.argv[1:] or [1, 2, 4, 8, 16, 64])]:
    ys = torch.from_numpy(np.stack([c.y] * B)).cuda()
    r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
    r.run(ys); torch.cuda.synchronize()
    acc = {}
    for _ in range(3):
        timer = {}
        r.run(ys, timer=timer); torch.cuda.synchronize()
        for k, v in Restorer.phase_times(timer).items():
            acc[k] = acc.get(k, 0.0) + v / 3
    tot = sum(acc.values())
    print(f"B={B:3d} ms/image: " + " ".join(f"{k} {v / B:.3f}" for k, v in acc.items()) + f" | total {tot / B:.3f}"
          f" -> {B * 1.048576 / (tot * 1e-3):.0f} MP/s", flush=True)
    del r, ys; torch.cuda.empty_cache()
