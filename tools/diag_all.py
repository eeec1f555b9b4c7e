import sys, time, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle'); sys.path.insert(0, '.')
from conftest import golden_inputs
from paper_1710_08124_b200 import synthetic, RestorationConfig, restore
models = {}
for P in (64, 100):
    m = synthetic.synthetic_gmm(200, P, 0, 0.95); models[P] = (m, synthetic.baseline_tree(m))
names = sys.argv[2:] or ["cfg1", "regular48", "gain64", "inpaint96", "deblur96", "sr96"]
for name in names:
    g, A, y, s8, s, P = golden_inputs(name)
    if not g["meta"]["use_tree"]: continue
    model, tree = models[P]
    for mode in sys.argv[1].split(","):
        cfg = RestorationConfig(sigma=s8, spacing=s, seed=0, trace=True, sampling=g["meta"]["sampling"])
        try:
            t0 = time.perf_counter()
            x, st = restore(y, A, model, tree, cfg, mode=mode)
            dt = time.perf_counter() - t0
        except Exception as e:
            print(name, mode, "ERROR", repr(e)[:300]); continue
        agree = [round(float(np.mean(r["selected"] == g["labels"][t])), 5) for t, r in enumerate(st.trace)]
        conv = [it.image_solve_converged for it in st.iterations]
        print(f"{name:10s} {mode:6s} agree {agree} rmse255 {255*np.sqrt(np.mean((x-g['x'])**2)):.3e} lam {st.lam:.10g} ref {float(g['lam']):.10g} conv {conv} ref {list(g['converged'])} rescored {st.rescored} wall {dt:.2f}s")
