"""Phase times (ms per restore of 64 x 1024^2) under a debug toggle:
python tools/phase_ab.py <fepll_debug_symbol> <value> [<value> ...]"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = 64
ys = np.stack([synthetic.baseline_case("cfg5", 1024, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", 1024).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
y = torch.from_numpy(ys).cuda()
fn = getattr(N.lib(), sys.argv[1]); fn.argtypes = [ctypes.c_int32]
r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
ref = None
for v in map(int, sys.argv[2:]):
    fn(v)
    x = r.run(y)[0].clone()
    if ref is None:
        ref = x
    same = bool(torch.equal(x, ref))
    best = {}
    for _ in range(3):
        timer = {}
        r.run(y, timer=timer)
        torch.cuda.synchronize()
        for k, t in Restorer.phase_times(timer).items():
            best[k] = min(best.get(k, 1e9), t)
    print(sys.argv[1], v, {k: round(t, 3) for k, t in best.items()}, "bitwise-equal to first:", same)
