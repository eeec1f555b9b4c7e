import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N
level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
c = synthetic.baseline_case("cfg5", 1024)
ys = np.stack([c.y] * B)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor")
y = torch.from_numpy(ys).cuda(); r.run(y)
buf = torch.zeros(148 * 64 * 16, dtype=torch.int64, device="cuda")
fn = N.lib().fepll_debug_ws_trace; fn.argtypes = [ctypes.c_void_p, ctypes.c_int32]
fn(buf.data_ptr(), level); r.run(y); torch.cuda.synchronize(); fn(None, -1)
tr = buf.view(148, 64, 16).cpu().numpy().astype(np.float64) / 1.965  # cycles -> ns
cta = 30
t0 = tr[cta, 0, 0]
print("ns relative to CTA start: p0=producers after a_empty wait, p1=stage stored, m2=MMA start, m3=issued, e4=acc ready, e5=epi math done, e6=routed")
for i in range(0, 14):
    row = tr[cta, i] - t0
    print(f"tile {i:2d}: p0 {row[0]:7.0f} p1 {row[1]:7.0f} | m2 {row[2]:7.0f} m3 {row[3]:7.0f} | 4 {row[4]:7.0f} 5 {row[5]:7.0f} 6 {row[6]:7.0f}")
d = lambda a, b: np.median((tr[:, 2:40, b] - tr[:, 2:40, a])[tr[:, 2:40, 2] > 0])
print("median ns: fill(p0->p1)", d(0, 1), "issue(m2->m3)", d(2, 3), "epi math(e4->e5)", d(4, 5), "route(e5->e6)", d(5, 6))
st = np.diff(tr[:, 2:40, 2], axis=1); print("MMA start spacing median ns", np.median(st[st > 0]))

iss = tr[:, 0:37, 7]; land = tr[:, 3:40, 0]; ok = (tr[:, 3:40, 0] > 0) & (iss > 0)
print("raw load latency (issue at i -> landed at i+3) median ns", np.median((land - iss)[ok]))
mm = tr[:, 0:36, 3]; iss4 = tr[:, 3:39, 7]; ok = (iss4 > 0) & (mm > 0)
print("refill issue(i+4 at iter i+1... ) minus MMA-issued(i): median ns", np.median((tr[:, 1:37, 7] - tr[:, 0:36, 3])[ok]))

print("producer: p1(i+1) -> raw_empty passed (slot 8 at i+1)", np.median((tr[:, 3:39, 8] - tr[:, 3:39, 1])[tr[:, 3:39, 8] > 0]))
print("producer: issue duration (slot 8 -> 7)", np.median((tr[:, 3:39, 7] - tr[:, 3:39, 8])[tr[:, 3:39, 8] > 0]))
print("MMA done (e4) - m3", np.median((tr[:, 3:39, 4] - tr[:, 3:39, 3])[tr[:, 3:39, 4] > 0]))

m = lambda a, b: np.median((tr[:, 3:39, b] - tr[:, 3:39, a])[tr[:, 3:39, b] > 0])
print("MMA loop: prev issued -> top", np.median((tr[:, 3:39, 10] - tr[:, 2:38, 3])[tr[:, 3:39, 10] > 0]),
      "acc_empty wait", m(10, 9), "lo_full wait", m(9, 2))
print("converter: raw_full passed (p0) - loader issued (slot 7)", m(7, 0))

g0 = tr[:, 63, 14] * 1.965; g1 = tr[:, 63, 15] * 1.965  # globaltimer ns (undo the cycle scaling)
ok = (g0 > 0) & (g1 > 0)
if ok.any():
    span = g1[ok] - g0[ok]
    print(f"CTA spans (globaltimer): mean {span.mean()/1e3:.1f} us, max {span.max()/1e3:.1f} us; "
          f"kernel start->last CTA end {(g1[ok].max() - g0[ok].min())/1e3:.1f} us; "
          f"first CTA end {(g1[ok].min() - g0[ok].min())/1e3:.1f} us")
