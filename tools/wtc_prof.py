"""Where the tcgen05 Wiener kernel waits: per-role wait cycles summed over a
launch (fepll_debug_wtc_prof), averaged over the CTAs, in microseconds.
Needs the library built with the counters: FEPLL_WTC_PROF=1 python -m
paper_1710_08124_b200.build --force (they are compiled out by default)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
tree = synthetic.baseline_tree(model)
r = Restorer(c.A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode="tensor",
             precision="fp32-state", options={"wiener_tc": 1})
y = torch.from_numpy(np.stack([c.y] * B)).cuda()
r.run(y)
buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
fn = N.lib().fepll_debug_wtc_prof
fn.argtypes = [ctypes.c_void_p]
r.start(y)
fn(buf.data_ptr())
r.iterate(0)
torch.cuda.synchronize()
fn(None)
p = buf.view(148, 32).cpu().numpy().astype(np.float64) / 1.9e3  # ~us at 1.9 GHz
names = ["loader: stage_free wait", "loader: loop total", "conv: raw_full wait", "conv: out_full wait",
         "conv: loop total", "mma: raw_full wait", "mma: lo_full wait", "mma: w_full wait",
         "mma: out_empty wait", "mma: leaf switches", "mma: loop total", "ep1: c_full wait", "ep1: loop total",
         "ep2a: raw_full wait", "ep2a: out_full wait", "ep2a: compute", "ep2a: loop total",
         "ep2b: raw_full wait", "ep2b: out_full wait", "ep2b: compute", "ep2b: loop total",
         "mma: first product issue", "mma: second product issue", "mma2: loop total"]
for k, nm in enumerate(names):
    print(f"{nm:28s} mean {p[:, k].mean():9.1f} us   min {p[:, k].min():9.1f}   max {p[:, k].max():9.1f}")
