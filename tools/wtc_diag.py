"""Diagnostic: fp32-state with the DMMA / tcgen05 Wiener step against the FP64
default on cfg5 images — label flips per iteration and RMSE (0..255)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
spec = synthetic.CONFIGS["cfg5"]
cases = [synthetic.baseline_case("cfg5", size, image_seed=i, noise_seed=1000 + i) for i in range(B)]
ys = np.stack([c.y for c in cases]).astype(np.float32).astype(np.float64)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
tree = synthetic.baseline_tree(model)
cfg = RestorationConfig(sigma=spec["sigma"], spacing=spec["spacing"], seed=0)
y = torch.from_numpy(ys).cuda()


def run(precision, opts):
    r = Restorer(cases[0].A, model, tree, cfg, batch=B, precision=precision, options=opts)
    r.start(y)
    labels, xs = [], []
    for t in range(len(r.betas)):
        r.iterate(t)
        labels.append(r.labels.view(B, r.n).cpu().numpy().copy())
        xs.append(r.x.cpu().numpy().astype(np.float64).copy())
    r.check_status()
    return labels, xs


ref_l, ref_x = run("fp64", {})
for name, prec, opts in [("fp32-state dmma", "fp32-state", {"wiener_tc": 0}),
                         ("fp32-state tcgen05", "fp32-state", {"wiener_tc": 1})]:
    l, x = run(prec, opts)
    for t in range(len(l)):
        flips = int((l[t] != ref_l[t]).sum())
        d = x[t] - ref_x[t]
        rm = 255 * np.sqrt((d ** 2).mean(axis=(1, 2)))
        print(f"{name} iter {t}: flips {flips} of {l[t].size}, rmse255 per image "
              f"{np.array2string(rm, precision=6)}, max|d|*255 {255 * np.abs(d).max():.4f}, "
              f"mean d*255 {255 * d.mean():+.2e}", flush=True)
