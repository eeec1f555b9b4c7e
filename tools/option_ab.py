"""Phase times (ms per restore) of a batch of cfg5 images under plan-option
values, and whether each value's image is bitwise-equal to the first's:
python tools/option_ab.py <option> <value> [<value> ...] [--batch B] [--size S] [--precision P]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic

ap = argparse.ArgumentParser()
ap.add_argument("option")
ap.add_argument("values", type=int, nargs="+")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
B, S = a.batch, a.size
ys = np.stack([synthetic.baseline_case("cfg5", S, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", S).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
tree = synthetic.baseline_tree(model)
y = torch.from_numpy(ys).cuda()
ref = None
for v in a.values:
    r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor",
                 options={a.option: v}, precision=a.precision)
    x = r.run(y)[0].clone()
    if ref is None:
        ref = x
    same = bool(torch.equal(x, ref))
    best = {}
    for _ in range(a.reps):
        timer = {}
        r.run(y, timer=timer)
        torch.cuda.synchronize()
        for k, t in Restorer.phase_times(timer).items():
            best[k] = min(best.get(k, 1e9), t)
    print(a.option, v, {k: round(t, 3) for k, t in best.items()}, "total", round(sum(best.values()), 3),
          "bitwise-equal to first:", same, flush=True)
    del r
    torch.cuda.empty_cache()
