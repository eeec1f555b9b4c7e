import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = 16; level = 6
c = synthetic.baseline_case("cfg5", 1024)
ys = np.stack([c.y] * B)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
y = torch.from_numpy(ys).cuda()
r.run(y)
buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
fn = N.lib().fepll_debug_ws_trace; fn.argtypes = [ctypes.c_void_p, ctypes.c_int32]
fl = N.lib().fepll_debug_ws_flags; fl.argtypes = [ctypes.c_int32]
for flags in [0, 1, 2, 3]:
    fl(flags); fn(buf.data_ptr(), level); r.run(y); torch.cuda.synchronize(); fn(None, -1)
    tr = buf.view(148, 64, 8).cpu().numpy().astype(np.float64)
    steps = np.diff(tr[:, :, 2], axis=1); mk = (tr[:, 1:, 2] > 0) & (tr[:, :-1, 2] > 0)
    iss = (tr[:, :, 3] - tr[:, :, 2])[tr[:, :, 2] > 0]
    print(f"flags={flags}: median MMA-start spacing {np.median(steps[mk])/1e3:.2f} us, issue {np.median(iss)/1e3:.2f} us")
fl(0)
fl(15); fn(buf.data_ptr(), level); r.run(y); torch.cuda.synchronize(); fn(None, -1); fl(0)
tr = buf.view(148, 64, 8).cpu().numpy().astype(np.float64)
t0 = tr[:, 0, 7].min()
for i in range(4, 16):
    row = (tr[20, i] - t0) / 1e3
    print(f"tile {i:2d}: prod {row[0]:7.2f}-{row[1]:7.2f} mma {row[2]:7.2f}-{row[3]:7.2f} mma-pre {row[4]:7.2f} acc_empty-done {row[5]:7.2f} mma-complete {row[6]:7.2f}")
