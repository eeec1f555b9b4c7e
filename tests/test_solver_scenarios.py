"""The reference's own restore tests (`pkg/tests/test_solver.py`) replayed
through the drop-in.

``tests/golden/solver_<scenario>.npz`` were written by
``oracle/make_golden.py`` executing the reference: its conftest model
builders, ``build_tree``, ``phantom_image`` and ``restore``.  The model and
tree arrive as the reference's FEPLLGM1 / FEPLLTR1 file bytes.

CPU tests: the oracle reproduces every stored run, and the drop-in raises
the reference's DataErrors (validation precedes any device work).  GPU
tests: the drop-in reproduces the stored labels, counters and images, and
the properties the reference's tests assert hold on its own trace records.
"""

import json
from dataclasses import replace

import numpy as np
import pytest
from conftest import GOLDEN

import fepll_oracle as O

SCENARIOS = ["basics", "exact16", "estimates16", "update16", "workers64", "profiles64", "tree16"]


def load(name, tmp_path):
    from paper_1710_08124_b200 import model_read, tree_read

    d = np.load(GOLDEN / f"solver_{name}.npz")
    g = {k: d[k] for k in d.files}
    g["meta"] = json.loads(str(g["meta"]))
    mp = tmp_path / f"{name}.gm"
    mp.write_bytes(g["model"].tobytes())
    g["model_obj"] = model_read(mp)
    g["tree_obj"] = None
    if "tree" in g:
        tp = tmp_path / f"{name}.tr"
        tp.write_bytes(g["tree"].tobytes())
        g["tree_obj"] = tree_read(tp)
    return g


def config(fields):
    from paper_1710_08124_b200 import RestorationConfig

    return RestorationConfig(**fields)


def rmse255(a, b):
    return 255.0 * float(np.sqrt(np.mean((np.asarray(a) - np.asarray(b)) ** 2)))


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("name", SCENARIOS)
def test_oracle_reproduces_reference_scenarios(name, tmp_path):
    g = load(name, tmp_path)
    for run, f in g["meta"]["runs"].items():
        c = config(f)
        y = g[f"y_{run}"]
        from paper_1710_08124_b200 import identity_operator

        x, st = O.restore(y, identity_operator(y.shape), g["model_obj"],
                          g["tree_obj"] if c.use_tree else None, sigma=c.sigma, spacing=c.spacing,
                          sampling=c.sampling, use_tree=c.use_tree, seed=c.seed, trace=c.trace)
        np.testing.assert_allclose(x, g[f"x_{run}"], rtol=0, atol=1e-12)
        cnt = np.array([st.patches, st.evals, st.sel_mults, st.est_mults]).T
        np.testing.assert_array_equal(cnt, g[f"counters_{run}"])
        if f"selected_{run}" in g:
            for t, rec in enumerate(st.trace):
                np.testing.assert_array_equal(rec["selected"], g[f"selected_{run}"][t])


def test_drop_in_validation_errors(tmp_path):
    """pkg/tests/test_solver.py:63-77 (tree required, full rank required,
    iteration count) — raised before any device work."""
    from paper_1710_08124_b200 import DataError, RestorationConfig, identity_operator, restore

    g = load("basics", tmp_path)
    y = g["y_seeded"]
    A = identity_operator(y.shape)
    with pytest.raises(DataError, match="tree"):
        restore(y, A, g["model_obj"], None, RestorationConfig(sigma=20.0))
    with pytest.raises(DataError, match="full-rank"):
        restore(y, A, g["model_obj"], None,
                RestorationConfig(sigma=20.0, use_tree=False, use_flat_tail=False))
    with pytest.raises(DataError):
        RestorationConfig(sigma=20.0, iterations=3).validate()
    with pytest.raises(DataError, match="observation shape"):
        restore(y[:40], A, g["model_obj"], g["tree_obj"], RestorationConfig(sigma=20.0))


# ------------------------------------------------------------------ GPU
def _restore(g, run, mode, **over):
    from paper_1710_08124_b200 import identity_operator, restore

    c = config(g["meta"]["runs"][run])
    if over:
        c = replace(c, **over)
    y = g[f"y_{run}"]
    return restore(y, identity_operator(y.shape), g["model_obj"], g["tree_obj"] if c.use_tree else None,
                   c, mode=mode)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["tensor", "exact"])
@pytest.mark.parametrize("name", SCENARIOS)
def test_drop_in_reproduces_reference_runs(name, mode, tmp_path):
    g = load(name, tmp_path)
    for run in g["meta"]["runs"]:
        x, st = _restore(g, run, mode, trace=True)
        assert rmse255(x, g[f"x_{run}"]) <= 1e-3
        assert float(np.abs(x - g[f"x_{run}"]).max()) <= 1e-10
        cnt = np.array([[it.patches, it.score_evaluations, it.selection_multiplies,
                         it.estimation_multiplies] for it in st.iterations])
        np.testing.assert_array_equal(cnt, g[f"counters_{run}"])
        if f"selected_{run}" in g:
            for t, rec in enumerate(st.trace):
                np.testing.assert_array_equal(rec["selected"], g[f"selected_{run}"][t])
        # trace records carry the reference's keys and the times its stats do
        rec = st.trace[0]
        assert set(rec) >= {"beta", "grid", "patches", "dc", "selected", "estimates", "x_tilde"}
        assert rec["grid"].positions.shape == (rec["patches"].shape[0], 2)
        assert set(st.iterations[0].times) >= {"grid", "extract", "select", "estimate", "reproject"}


@pytest.mark.gpu
def test_basics_properties(tmp_path):
    """pkg/tests/test_solver.py:50-84: noiseless pass-through, same seed
    bit-identical, output not clamped."""
    g = load("basics", tmp_path)
    x, _ = _restore(g, "noiseless", "tensor")
    assert np.sqrt(np.mean((x - g["y_noiseless"]) ** 2)) < 1e-3
    a, _ = _restore(g, "seeded", "tensor")
    b, _ = _restore(g, "seeded", "tensor")
    assert np.array_equal(a, b)
    x, _ = _restore(g, "unclamped", "tensor")
    assert x.max() > 1.0


@pytest.mark.gpu
def test_exact_profile_selections_are_exact_argmin(tmp_path):
    """pkg/tests/test_solver.py:87-102 on the drop-in's own trace: labels =
    argmin of the exact (tail-free, full-rank) scores of the traced patches."""
    g = load("exact16", tmp_path)
    _, st = _restore(g, "exact", "tensor")
    comps = g["model_obj"].components
    assert len(st.trace) == 5
    for rec in st.trace:
        beta = rec["beta"]
        Z = rec["patches"]
        exact = np.empty((Z.shape[0], len(comps)))
        for k, c in enumerate(comps):
            nu = c.kept_eigenvalues + 1.0 / beta
            coeffs = Z @ c.kept_basis
            exact[:, k] = -2.0 * np.log(c.weight) + np.log(nu).sum() + np.square(coeffs) @ (1.0 / nu)
        np.testing.assert_array_equal(rec["selected"], np.argmin(exact, axis=1))


@pytest.mark.gpu
def test_patch_estimates_minimize_surrogate(tmp_path):
    """pkg/tests/test_solver.py:104-119: beta (zhat - z) + Sigma^-1 zhat = 0
    for the drop-in's traced estimates."""
    g = load("estimates16", tmp_path)
    _, st = _restore(g, "run", "tensor")
    rec = st.trace[-1]
    beta = rec["beta"]
    rng = np.random.default_rng(12)
    for i in rng.choice(rec["patches"].shape[0], 40, replace=False):
        k = rec["selected"][i]
        cov = g["model_obj"].components[k].covariance()
        zt, zh = rec["patches"][i], rec["estimates"][i]
        resid = beta * (zh - zt) + np.linalg.solve(cov, zh)
        assert np.abs(resid).max() < 1e-6 * max(1.0, beta * np.abs(zt).max())


@pytest.mark.gpu
def test_image_update_optimality(tmp_path):
    """pkg/tests/test_solver.py:121-134."""
    g = load("update16", tmp_path)
    x, st = _restore(g, "run", "tensor")
    rec = st.trace[-1]
    bs2 = rec["beta"] * (20.0 / 255.0) ** 2
    rhs = g["y_run"] + bs2 * rec["x_tilde"]
    resid = x + bs2 * x - rhs
    assert np.linalg.norm(resid) <= 1e-6 * np.linalg.norm(rhs)


@pytest.mark.gpu
def test_worker_count_invariance(tmp_path):
    """pkg/tests/test_solver.py:137-148: the device path ignores the CPU
    thread-pool size; every worker count gives the reference's image."""
    g = load("workers64", tmp_path)
    base, _ = _restore(g, "w1", "tensor")
    assert float(np.abs(base - g["x_w1"]).max()) <= 1e-10
    for w in (2, 8):
        x, _ = _restore(g, "w1", "tensor", workers=w)
        assert np.array_equal(base, x)


@pytest.mark.gpu
def test_profile_counter_ratio(tmp_path):
    """pkg/tests/test_solver.py:152-170: spacing-6 jittered subsampling cuts
    the selection and estimation multiplies ~36x."""
    g = load("profiles64", tmp_path)
    _, none = _restore(g, "none", "tensor")
    _, sub = _restore(g, "subsample", "tensor")
    ratio = none.total_selection_multiplies / sub.total_selection_multiplies
    assert abs(ratio - 36.0) <= 3.6
    est = none.total_estimation_multiplies / sub.total_estimation_multiplies
    assert abs(est - 36.0) <= 3.6


@pytest.mark.gpu
def test_tree_profile_reduces_evaluations(tmp_path):
    """pkg/tests/test_solver.py:172-187."""
    g = load("tree16", tmp_path)
    K = len(g["model_obj"].components)
    _, tr = _restore(g, "tree", "tensor")
    _, flat = _restore(g, "no-tree", "tensor")
    assert tr.total_score_evaluations / tr.total_patches < K
    assert flat.total_score_evaluations / flat.total_patches == K
