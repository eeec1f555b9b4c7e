import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = int(sys.argv[1]); level = int(sys.argv[2])
c = synthetic.baseline_case("cfg5", 1024)
ys = np.stack([c.y] * B)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
y = torch.from_numpy(ys).cuda()
r.run(y)
buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
fn = N.lib().fepll_debug_ws_trace; fn.argtypes = [ctypes.c_void_p, ctypes.c_int32]
fn(buf.data_ptr(), level); r.run(y); torch.cuda.synchronize(); fn(None, -1)
tr = buf.view(148, 64, 8).cpu().numpy().astype(np.float64)
t0 = tr[:, 0, 7].min()
cta = 10
print("slots: p0 p1 m2 m3 e4 e5 e6 (us rel. kernel start)")
for i in range(0, 24):
    row = (tr[cta, i] - t0) / 1e3
    print(f"tile {i:2d}: prod {row[0]:7.2f}-{row[1]:7.2f} mma {row[2]:7.2f}-{row[3]:7.2f} epi {row[4]:7.2f}-{row[5]:7.2f}-{row[6]:7.2f}")
