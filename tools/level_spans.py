"""Per-level timeline of the ws2 tree-level kernels inside one CUDA-graph
replay of a cfg5 batch restore: CTA entry, prologue end and CTA end
(globaltimer), and the gaps between consecutive levels.
python tools/level_spans.py [B] [size]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic, _native as N

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ys = np.stack([synthetic.baseline_case("cfg5", S, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", S).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
tree = synthetic.baseline_tree(model)
y = torch.from_numpy(ys).cuda()
r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B)
r.run(y)
D = 16
buf = torch.zeros(D * 148 * 4 + 2 * D, dtype=torch.int64, device="cuda")
buf[D * 148 * 4::2] = -1  # atomic-min slots (as uint64: ~0)
N.lib().fepll_debug_level_spans(buf.data_ptr())
r.capture(y)
r.replay()
torch.cuda.synchronize()
buf.zero_()
buf[D * 148 * 4::2] = -1
r.replay()
torch.cuda.synchronize()
N.lib().fepll_debug_level_spans(None)
raw = buf.cpu().numpy()
rs = raw[D * 148 * 4:].reshape(D, 2).astype(np.float64)
t = raw[:D * 148 * 4].reshape(D, 148, 4).astype(np.float64)
levels = [d for d in range(D) if (t[d, :, 0] > 0).any()]
t0 = t[levels[0], :, 0][t[levels[0], :, 0] > 0].min()
prev_end = None
tot = 0.0
for d in levels:
    e, p, x = (t[d, :, k] for k in range(3))
    ok = e > 0
    e, p, x = e[ok] - t0, p[ok] - t0, x[ok] - t0
    span = x.max() - e.min()
    tot += span
    gap = (e.min() - prev_end) if prev_end is not None else 0.0
    print(f"level {d}: gap from previous {gap/1e3:6.1f} us | entry {e.min()/1e3:8.1f}..{e.max()/1e3:8.1f} "
          f"prologue {np.median(p - e)/1e3:5.1f} us | work {np.median(x - p)/1e3:6.1f} us (min {np.min(x - p)/1e3:6.1f} max {np.max(x - p)/1e3:6.1f}) "
          f"| first end {x.min()/1e3 - e.min()/1e3:6.1f} last end {span/1e3:6.1f} us")
    prev_end = x.max()
    if rs[d, 1] > 0:
        r0, r1 = rs[d, 0] - t0, rs[d, 1] - t0
        print(f"   re-score: start {(r0 - prev_end)/1e3:5.1f} us after the level, runs {(r1 - r0)/1e3:5.1f} us")
        prev_end = r1
print(f"levels {len(levels)}: sum of kernel spans {tot/1e3:.1f} us, first entry -> last end "
      f"{(prev_end)/1e3:.1f} us")
# per-CTA work of the last level (CTAs own contiguous tile ranges in node order)
d = levels[-1]
e, p, x = (t[d, :, k] for k in range(3))
wk = (x - p) / 1e3
order = np.argsort(-wk)
print("slowest CTAs of level", d, [(int(i), round(float(wk[i]), 1)) for i in order[:12]])
print("work by CTA block of 16:", [round(float(np.mean(wk[i:i + 16])), 1) for i in range(0, 148, 16)])
