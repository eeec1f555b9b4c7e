"""A/B: dc restored in the Wiener epilogue (default) vs added by the cover gather."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = 64
ys = np.stack([synthetic.baseline_case("cfg5", 1024, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", 1024).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
y = torch.from_numpy(ys).cuda()
fn = N.lib().fepll_debug_wiener_dc; fn.argtypes = [ctypes.c_int32]
r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
ref = None
for on in (1, 0, 1, 0):
    fn(on)
    r._agg_dc = None if on else r.dc
    x = r.run(y)[0].clone()
    ref = x if ref is None else ref
    best = {}
    for _ in range(3):
        timer = {}
        r.run(y, timer=timer)
        torch.cuda.synchronize()
        for k, t in Restorer.phase_times(timer).items():
            best[k] = min(best.get(k, 1e9), t)
    print("wiener_dc", on, {k: round(t, 3) for k, t in best.items()}, "equal:", bool(torch.equal(x, ref)))
