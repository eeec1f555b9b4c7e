"""Select-phase cost vs the certification guard (more re-scoring as it grows)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
B = 64
ys = np.stack([synthetic.baseline_case("cfg5", 1024, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", 1024).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
y = torch.from_numpy(ys).cuda()
for g in [2.0 ** -e for e in (sys.argv[1:] and map(int, sys.argv[1:]) or (16, 15, 14, 13))]:
    r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor", guard=g)
    r.run(y)
    best = None
    for _ in range(3):
        timer = {}
        r.run(y, timer=timer)
        torch.cuda.synchronize()
        ph = Restorer.phase_times(timer)
        best = ph if best is None or ph["select"] < best["select"] else best
    r.rescored.zero_(); r.run(y)
    frac = float(r.rescored.sum().item()) / (r.batch * r.n * 7)
    print(f"guard 2^{int(np.log2(g))}: select {best['select']:.3f} ms, rescored {frac:.2e}")
