"""Generate the golden fixtures in ``tests/golden/`` by EXECUTING the
reference package (``/root/reference/pkg/src``) — build-container only.

Outputs (all small):

* ``tree_partitions_P64.json`` / ``tree_partitions_P100.json`` — the level
  partitions of ``fepll.tree.build_tree(synthetic_gmm(P), seed=0)`` plus
  the sha256 of the reference ``tree_write`` bytes;
* ``restore_<case>.npz`` — reference ``restore(..., trace=True)`` results:
  lambda, betas, per-iteration selected labels, counters, CG flags, and the
  final image;
* ``grids.npz`` — reference ``jittered_grid`` anchors for a sweep of
  (H, W, P, s, seed, t), including spacing 1 and half == 0 cases;
* ``solver_<scenario>.npz`` — the scenarios of the reference's own restore
  tests (``pkg/tests/test_solver.py``): model and tree files written by the
  reference (FEPLLGM1 / FEPLLTR1 bytes), its phantom image, observations,
  restored images, per-iteration labels and counters.

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--solver-only]
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import fepll  # noqa: E402  (the reference)
from fepll import operators as rops  # noqa: E402
from fepll.gmm import FlatTailComponent as RComp, GmmModel as RModel  # noqa: E402
from fepll.patches import jitter_rng, jittered_grid  # noqa: E402
from fepll.solver import RestorationConfig, restore  # noqa: E402
from fepll.tree import build_tree, tree_write  # noqa: E402

from paper_1710_08124_b200 import synthetic  # noqa: E402
from paper_1710_08124_b200.tree import tree_partitions  # noqa: E402

OUT = ROOT / "tests" / "golden"

CASES = {
    # name: (config key, size, overrides)
    "cfg1": dict(cfg="cfg1", size=None),
    "deblur96": dict(cfg="cfg3", size=96),
    "inpaint96": dict(cfg="cfg4a", size=96),
    "sr96": dict(cfg="cfg4b", size=96),
    "gain64": dict(cfg="gain", size=64),
    "notree64": dict(cfg="cfg1", size=64, use_tree=False),
    "regular48": dict(cfg="cfg1", size=48, sampling="regular", spacing=3),
}


def ref_model(m):
    return RModel(m.patch_dim, [RComp(c.weight, c.kept_basis, c.kept_eigenvalues, c.tail_value)
                                for c in m.components], m.rho)


def case_inputs(spec):
    if spec["cfg"] == "gain":
        H = spec["size"]
        img = synthetic.synthetic_image(H, H, 0)
        g = rops.radial_gain_map((H, H), 0.6)
        A = rops.gain_operator(g)
        y = g * (img + 5.0 * np.random.default_rng(1).standard_normal((H, H))) / 255.0
        return A, y, 5.0, 4, 64
    c = synthetic.baseline_case(spec["cfg"], spec["size"])
    A = c.A
    RA = {"identity": lambda: rops.identity_operator(A.input_dims),
          "convolution": lambda: rops.convolution_operator(A.kernel, A.input_dims),
          "mask": lambda: rops.mask_operator(A.pixel_map),
          "decimate": lambda: rops.decimate_operator(A.factor, A.input_dims, A.kernel)}[A.kind]()
    return RA, c.y, c.sigma8, c.spacing, c.patch_dim


def _noisy(img, sigma8, seed):
    """pkg/tests/test_solver.py:23-25"""
    rng = np.random.default_rng(seed)
    return img + (sigma8 / 255.0) * rng.standard_normal(img.shape)


# The scenarios of the reference's own restore tests (pkg/tests/
# test_solver.py), with the models, trees and phantom images built by the
# reference (its conftest builders, build_tree, phantom_image).  Each run
# stores the reference's outputs so the GPU drop-in replays them exactly.
SOLVER_SCENARIOS = {
    # TestRestoreBasics (:44-84): 5-component P=64 model flattened at 0.95 + tree
    "basics": dict(model=(5, 64, 0), flatten=0.95, tree=dict(seed=0), image=(48, 1), runs={
        "noiseless": dict(noise=None, cfg=dict(sigma=0.0, spacing=4, seed=0)),
        "seeded": dict(noise=(20, 2), cfg=dict(sigma=20.0, seed=3)),
        "unclamped": dict(noise="plus_half", cfg=dict(sigma=0.0, spacing=4, seed=0))}),
    # TestAccelerationSoundness.test_exact_profile_selections (:87-102)
    "exact16": dict(model=(6, 16, 6), flatten=None, tree=None, image=(24, 7), runs={
        "exact": dict(noise=(20, 8), cfg=dict(sigma=20.0, use_tree=False, use_flat_tail=False,
                                              spacing=1, sampling="regular", trace=True))}),
    # test_patch_estimates_minimize_surrogate (:104-119)
    "estimates16": dict(model=(4, 16, 9), flatten=0.9, tree=dict(levels=(2, 1), seed=0), image=(24, 10),
                        runs={"run": dict(noise=(20, 11), cfg=dict(sigma=20.0, spacing=3, trace=True, seed=1))}),
    # test_image_update_optimality (:121-134)
    "update16": dict(model=(4, 16, 13), flatten=None, tree=None, image=(24, 14), runs={
        "run": dict(noise=(20, 15), cfg=dict(sigma=20.0, use_tree=False, use_flat_tail=False,
                                            spacing=1, sampling="regular", trace=True))}),
    # TestWorkers (:137-148)
    "workers64": dict(model=(6, 64, 16), flatten=0.9, tree=dict(seed=0), image=(96, 17), runs={
        "w1": dict(noise=(20, 18), cfg=dict(sigma=20.0, spacing=1, sampling="regular", seed=5)),
        "w8": dict(noise=(20, 18), cfg=dict(sigma=20.0, spacing=1, sampling="regular", seed=5,
                                            workers=8))}),
    # TestCompareProfiles.test_counter_ratio_and_quality_rows (:152-170)
    "profiles64": dict(model=(5, 64, 19), flatten=None, tree=None, image=(128, 20), runs={
        "none": dict(noise=(20, 21), cfg=dict(sigma=20.0, seed=0, use_flat_tail=False, use_tree=False,
                                              spacing=1, sampling="regular")),
        "subsample": dict(noise=(20, 21), cfg=dict(sigma=20.0, seed=0, use_flat_tail=False,
                                                   use_tree=False))}),
    # test_tree_profile_reduces_evaluations (:172-187): tree of the full-rank
    # model at rho 1 (solver.py:292-311 _profile_assets)
    "tree16": dict(model=(20, 16, 22), flatten=None, tree=dict(seed=0, rho=1.0), image=(64, 23), runs={
        "tree": dict(noise=(20, 24), cfg=dict(sigma=20.0, spacing=2, seed=0, use_flat_tail=False)),
        "no-tree": dict(noise=(20, 24), cfg=dict(sigma=20.0, spacing=2, seed=0, use_flat_tail=False,
                                                 use_tree=False))}),
}


def solver_scenarios():
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import synthetic_model  # the reference's own builder
    from fepll.model_io import model_write
    from fepll.operators import identity_operator
    from fepll.phantoms import phantom_image

    for name, sc in SOLVER_SCENARIOS.items():
        K, P, mseed = sc["model"]
        model = synthetic_model(K, P, seed=mseed)
        if sc["flatten"] is not None:
            model = model.flatten(sc["flatten"])
        tree = None
        if sc["tree"] is not None:
            tkw = dict(sc["tree"])
            tree = build_tree(model, tkw.pop("levels", None), seed=tkw.pop("seed"), **tkw)
        mpath, tpath = Path(f"/tmp/golden_{name}.gm"), Path(f"/tmp/golden_{name}.tr")
        model_write(model, mpath)
        out = {"model": np.frombuffer(mpath.read_bytes(), np.uint8)}
        if tree is not None:
            tree_write(tree, tpath)
            out["tree"] = np.frombuffer(tpath.read_bytes(), np.uint8)
        H, iseed = sc["image"]
        img = phantom_image(H, H, iseed)
        out["img"] = img
        meta = {"runs": {}}
        for run, spec in sc["runs"].items():
            if spec["noise"] is None:
                y = img.copy()
            elif spec["noise"] == "plus_half":
                y = img + 0.5
            else:
                y = _noisy(img, *spec["noise"])
            cfg = RestorationConfig(**spec["cfg"])
            x, st = restore(y, identity_operator(y.shape), model, tree if cfg.use_tree else None, cfg)
            out[f"y_{run}"] = y
            out[f"x_{run}"] = x
            if cfg.trace:
                out[f"selected_{run}"] = np.stack([r["selected"] for r in st.trace]).astype(np.int16)
            out[f"counters_{run}"] = np.array([[it.patches, it.score_evaluations, it.selection_multiplies,
                                                it.estimation_multiplies] for it in st.iterations],
                                              dtype=np.int64)
            meta["runs"][run] = spec["cfg"]
        out["meta"] = json.dumps(meta)
        np.savez_compressed(OUT / f"solver_{name}.npz", **out)
        print("scenario", name, {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    if "--solver-only" in sys.argv:
        solver_scenarios()
        return
    models, trees = {}, {}
    for P in (64, 100):
        m = synthetic.synthetic_gmm(200, P, 0, 0.95)
        rm = ref_model(m)
        t = build_tree(rm, seed=0)
        path = Path(f"/tmp/golden_tree_{P}.bin")
        tree_write(t, path)
        digest = hashlib.sha256(path.read_bytes()).hexdigest()
        (OUT / f"tree_partitions_P{P}.json").write_text(json.dumps(
            {"source": "fepll.tree.build_tree(synthetic_gmm(200, P, 0, 0.95), seed=0)",
             "reference_tree_sha256": digest, "partitions": tree_partitions(t)}))
        models[P], trees[P] = rm, t
        print("tree", P, digest[:16])

    for name, spec in CASES.items():
        A, y, s8, s, P = case_inputs(spec)
        cfg = RestorationConfig(sigma=s8, spacing=spec.get("spacing", s), seed=0, trace=True,
                                use_tree=spec.get("use_tree", True),
                                sampling=spec.get("sampling", "jittered"))
        x, st = restore(y, A, models[P], trees[P] if cfg.use_tree else None, cfg)
        labels = np.stack([r["selected"] for r in st.trace]).astype(np.int16)
        np.savez_compressed(
            OUT / f"restore_{name}.npz",
            lam=st.lam, betas=np.array([it.beta for it in st.iterations]),
            labels=labels, x=x, y=y,
            patches=np.array([it.patches for it in st.iterations]),
            evals=np.array([it.score_evaluations for it in st.iterations]),
            sel_mults=np.array([it.selection_multiplies for it in st.iterations]),
            est_mults=np.array([it.estimation_multiplies for it in st.iterations]),
            converged=np.array([it.image_solve_converged for it in st.iterations]),
            residual=np.array([it.image_solve_residual for it in st.iterations]),
            xt_sha=np.array([hashlib.sha256(r["x_tilde"].tobytes()).hexdigest() for r in st.trace]),
            meta=json.dumps({"cfg": spec["cfg"], "size": spec["size"], "sigma": s8,
                             "spacing": cfg.spacing, "patch_dim": P, "kind": A.kind,
                             "use_tree": cfg.use_tree, "sampling": cfg.sampling}))
        print(name, A.kind, x.shape, "lam", st.lam, "patches", st.iterations[0].patches)

    sweep = []
    for (H, W, P, s) in [(64, 64, 64, 6), (41, 53, 64, 3), (256, 256, 64, 4), (96, 80, 100, 6),
                         (40, 40, 64, 8), (33, 47, 64, 1), (512, 512, 64, 2), (510, 510, 100, 6),
                         (37, 29, 100, 4), (1024, 1024, 64, 4)]:
        for seed in (0, 3, 2 ** 40 + 7):
            for t in (0, 1, 4):
                g = jittered_grid(H, W, P, s, jitter_rng(seed, t))
                sweep.append(((H, W, P, s, seed, t), g.positions.astype(np.int32)))
    keys = np.array([k for k, _ in sweep], dtype=np.uint64)
    small = {f"pos_{i}": p for i, (_, p) in enumerate(sweep) if p.shape[0] <= 20000}
    shas = np.array([hashlib.sha256(p.astype("<i4").tobytes()).hexdigest() for _, p in sweep])
    np.savez_compressed(OUT / "grids.npz", keys=keys, sha=shas, **small)
    print("grids", len(sweep))
    solver_scenarios()


if __name__ == "__main__":
    main()
