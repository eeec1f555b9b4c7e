"""Per-tile timeline of the Wiener kernel (clock64 stamps, CTA 30)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
y = torch.from_numpy(np.stack([c.y] * B)).cuda(); r.run(y)
buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
fn = N.lib().fepll_debug_wiener_trace; fn.argtypes = [ctypes.c_void_p]
fn(buf.data_ptr()); r.start(y); r.iterate(0); torch.cuda.synchronize(); fn(None)
tr = buf.view(148, 64, 8).cpu().numpy().astype(np.float64) / 1.965
print("ns per tile (median over CTAs, tiles 2..40): 0 top, 1 rows landed+sync, 2 next issued(+U), 3 phase1, 4 phase2, 5 written")
d = np.diff(tr[:, 2:40, :6], axis=2)
print("segments:", np.round(np.median(d, axis=(0, 1))).tolist())
print("tile period:", np.median(np.diff(tr[:, 2:40, 0], axis=1)))
