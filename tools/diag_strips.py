import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1710_08124_b200 import RestorationConfig, identity_operator, restore, synthetic
from paper_1710_08124_b200.strips import restore_strips_single_process, strip_specs
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
H, W, world, s = 160, 96, 3, 4
img = synthetic.synthetic_image(H, W, 3) / 255.0
y = img + (25.0 / 255.0) * np.random.default_rng(5).standard_normal((H, W))
print([ (sp.r0, sp.r1, sp.slab_lo, sp.slab_hi, sp.a_lo, sp.a_hi) for sp in strip_specs(H, W, 64, s, 2, world)])
for iters in (1, 2, 5):
    for mode in ("exact", "tensor"):
        cfg = RestorationConfig(sigma=25.0, spacing=s, seed=2, iterations=iters, beta_multipliers=(1.0, 4.0, 8.0, 16.0, 32.0)[:iters])
        xf, _ = restore(y, identity_operator((H, W)), model, tree, cfg, mode=mode)
        xs = restore_strips_single_process(y, model, tree, cfg, world, mode=mode)
        d = np.abs(xf - xs)
        rows = np.where(d.max(axis=1) > 0)[0]
        print(iters, mode, "maxdiff", d.max(), "rows", rows[:20], len(rows))
