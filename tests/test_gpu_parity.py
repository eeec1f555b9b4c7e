"""Device path vs the golden vectors and the live oracle (needs a B200)."""

import numpy as np
import pytest
from conftest import golden_inputs

import fepll_oracle as O

pytestmark = pytest.mark.gpu


def _rmse255(a, b):
    return 255.0 * float(np.sqrt(np.mean((np.asarray(a) - np.asarray(b)) ** 2)))


def _psnr(x, ref):
    mse = float(np.mean((np.clip(x, 0, 1) - ref) ** 2))
    return 10 * np.log10(1.0 / mse)


@pytest.mark.parametrize("mode", ["exact", "tensor"])
@pytest.mark.parametrize("name", ["cfg1", "gain64", "regular48"])
def test_restore_matches_golden(name, mode, models):
    from paper_1710_08124_b200 import RestorationConfig, restore

    g, A, y, s8, s, P = golden_inputs(name)
    meta = g["meta"]
    model, tree = models[P]
    cfg = RestorationConfig(sigma=s8, spacing=s, seed=0, trace=True, sampling=meta["sampling"])
    x, st = restore(y, A, model, tree, cfg, mode=mode)
    agree = [float(np.mean(rec["selected"] == g["labels"][t])) for t, rec in enumerate(st.trace)]
    assert min(agree) >= 0.999, agree
    assert _rmse255(x, g["x"]) <= 1e-3
    if mode == "exact":
        assert min(agree) == 1.0
        assert [it.score_evaluations for it in st.iterations] == list(g["evals"])
        assert [it.selection_multiplies for it in st.iterations] == list(g["sel_mults"])
        assert [it.estimation_multiplies for it in st.iterations] == list(g["est_mults"])
