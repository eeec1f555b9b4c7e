import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
B = int(sys.argv[1]); level = int(sys.argv[2])
ys = np.stack([synthetic.baseline_case("cfg5", 1024, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", 1024).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
y = torch.from_numpy(ys).cuda()
r.run(y)
buf = torch.zeros(148 * 64 * 8, dtype=torch.int64, device="cuda")
fn = N.lib().fepll_debug_ws_trace; fn.argtypes = [ctypes.c_void_p, ctypes.c_int32]
fn(buf.data_ptr(), level)
r.run(y)  # every iteration overwrites; last iteration's level remains
torch.cuda.synchronize()
fn(None, -1)
tr = buf.view(148, 64, 8).cpu().numpy().astype(np.float64)
t0 = tr[:, 0, 7].min()
for cta in [0, 37, 74, 147]:
    print("CTA", cta, "start", (tr[cta, 0, 7] - t0) / 1e3)
    for i in range(0, 64, 8):
        row = tr[cta, i]
        if row[0] == 0: break
        print(f"  tile {i:2d}: prod {(row[0]-t0)/1e3:8.2f}-{(row[1]-t0)/1e3:8.2f}  mma {(row[2]-t0)/1e3:8.2f}-{(row[3]-t0)/1e3:8.2f}  epi {(row[4]-t0)/1e3:8.2f}-{(row[5]-t0)/1e3:8.2f}-{(row[6]-t0)/1e3:8.2f} us")
valid = tr[:, 1:, 0] > 0
d = np.diff(tr[:, :, 2], axis=1)[valid[:, :]] if False else None
pp = (tr[:, :, 1] - tr[:, :, 0]); mm = (tr[:, :, 3] - tr[:, :, 2]); e1 = tr[:, :, 5] - tr[:, :, 4]; e2 = tr[:, :, 6] - tr[:, :, 5]
m = tr[:, :, 0] > 0
print("median us: producer", np.median(pp[m]) / 1e3, "mma issue", np.median(mm[m]) / 1e3, "epi compute", np.median(e1[m]) / 1e3, "epi route", np.median(e2[m]) / 1e3)
steps = np.diff(tr[:, :, 2], axis=1); mk = (tr[:, 1:, 2] > 0) & (tr[:, :-1, 2] > 0)
print("median MMA-start spacing us", np.median(steps[mk]) / 1e3)
