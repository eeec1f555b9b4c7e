"""Small driver for ncu captures: one restore of B synthetic 1024^2 images."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_08124_b200 import RestorationConfig, Restorer, synthetic
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
mode = sys.argv[3] if len(sys.argv) > 3 else "tensor"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[5].split(",")) if len(sys.argv) > 5 and sys.argv[5] else {}
precision = sys.argv[6] if len(sys.argv) > 6 else "fp64"
ys = np.stack([synthetic.baseline_case("cfg5", size, image_seed=i, noise_seed=1000 + i).y for i in range(B)])
A = synthetic.baseline_case("cfg5", size).A
model = synthetic.synthetic_gmm(200, 64, 0, 0.95); tree = synthetic.baseline_tree(model)
r = Restorer(A, model, tree, RestorationConfig(sigma=25.0, spacing=4, seed=0), batch=B, mode=mode, options=opts,
             precision=precision)
y = torch.from_numpy(ys).cuda()
for _ in range(reps):
    r.run(y)
torch.cuda.synchronize()
print("ok", r.counters()[0])
