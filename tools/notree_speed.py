"""No-tree (exhaustive) profile throughput: tcgen05 chunked scan vs FP64 scan."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = synthetic.baseline_case("cfg5", 1024)
model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
ys = torch.from_numpy(np.stack([c.y] * B)).cuda()
for mode in ("tensor", "exact"):
    r = Restorer(c.A, model, None, RestorationConfig(sigma=25.0, spacing=4, seed=0, use_tree=False), batch=B, mode=mode)
    r.run(ys); torch.cuda.synchronize()
    timer = {}
    t0 = time.perf_counter(); r.run(ys, timer=timer); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ph = Restorer.phase_times(timer)
    print(mode, f"{B * 1.048576 / dt:.1f} MP/s", {k: round(v, 2) for k, v in ph.items()},
          "rescored/level", [int(v) for v in r.rescored.sum(dim=1).cpu()][:5], flush=True)
