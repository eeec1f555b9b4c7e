import sys, time, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle'); sys.path.insert(0, '.')
from conftest import golden_inputs
from paper_1710_08124_b200 import synthetic, RestorationConfig, restore
models = {}
for P in (64, 100):
    m = synthetic.synthetic_gmm(200, P, 0, 0.95); models[P] = (m, synthetic.baseline_tree(m))
for name in sys.argv[1:] or ["cfg1", "regular48"]:
    g, A, y, s8, s, P = golden_inputs(name)
    model, tree = models[P]
    cfg = RestorationConfig(sigma=s8, spacing=s, seed=0, trace=True, sampling=g["meta"]["sampling"])
    x, st = restore(y, A, model, tree, cfg, mode="tensor")
    agree = [float(np.mean(r["selected"] == g["labels"][t])) for t, r in enumerate(st.trace)]
    print(name, "agree", agree, "rmse255", 255*np.sqrt(np.mean((x-g["x"])**2)), "rescored", st.rescored, "patches", [it.patches for it in st.iterations])
