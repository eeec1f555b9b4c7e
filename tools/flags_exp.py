import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = 16
c = synthetic.baseline_case("cfg5", 1024)
ys = np.stack([c.y] * B)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
y = torch.from_numpy(ys).cuda()
fl = N.lib().fepll_debug_ws_flags; fl.argtypes = [ctypes.c_int32]
r.run(y)
for flags in [0, 1, 2, 3]:
    fl(flags)
    for _ in range(2): r.run(y)
    timer = {}
    r.run(y, timer=timer); torch.cuda.synchronize()
    print(flags, {k: round(v, 2) for k, v in Restorer.phase_times(timer).items()})
fl(0)
