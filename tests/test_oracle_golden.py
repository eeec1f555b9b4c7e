"""Pin the CPU oracle against golden vectors produced by the reference
package itself (oracle/make_golden.py).  CPU only."""

import hashlib
import json

import numpy as np
import pytest
from conftest import GOLDEN, golden_inputs

import fepll_oracle as O
from paper_1710_08124_b200 import synthetic
from paper_1710_08124_b200.model_io import tree_write
from paper_1710_08124_b200.patches import jitter_rng, jittered_grid

CASES = ["cfg1", "deblur96", "inpaint96", "sr96", "gain64", "notree64", "regular48"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference(name, models):
    g, A, y, s8, s, P = golden_inputs(name)
    model, tree = models[P]
    meta = g["meta"]
    x, st = O.restore(y, A, model, tree, sigma=s8, spacing=s, seed=0,
                      use_tree=meta["use_tree"], sampling=meta["sampling"], trace=True)
    assert st.lam == pytest.approx(float(g["lam"]), rel=1e-12)
    np.testing.assert_allclose(st.betas, g["betas"], rtol=1e-12)
    for t, rec in enumerate(st.trace):
        np.testing.assert_array_equal(rec["selected"], g["labels"][t])
    assert st.patches == list(g["patches"])
    assert st.evals == list(g["evals"])
    assert st.sel_mults == list(g["sel_mults"])
    assert st.est_mults == list(g["est_mults"])
    assert st.converged == list(g["converged"])
    np.testing.assert_allclose(x, g["x"], rtol=0, atol=1e-12)


def test_golden_inputs_regenerate(models):
    # the product-side generators rebuild the exact observations the
    # reference was run on
    for name in ["cfg1", "inpaint96", "sr96"]:
        g, A, y, *_ = golden_inputs(name)
        meta = g["meta"]
        c = synthetic.baseline_case(meta["cfg"], meta["size"])
        np.testing.assert_array_equal(c.y, g["y"])


@pytest.mark.parametrize("P", [64, 100])
def test_tree_rebuild_matches_reference_bytes(P, models, tmp_path):
    _, tree = models[P]
    path = tmp_path / "t.bin"
    tree_write(tree, path)
    ref = json.loads((GOLDEN / f"tree_partitions_P{P}.json").read_text())["reference_tree_sha256"]
    assert hashlib.sha256(path.read_bytes()).hexdigest() == ref


def test_grids_match_reference():
    d = np.load(GOLDEN / "grids.npz")
    for i, key in enumerate(d["keys"]):
        H, W, P, s, seed, t = (int(v) for v in key)
        pos = jittered_grid(H, W, P, s, jitter_rng(seed, t)).positions.astype("<i4")
        assert hashlib.sha256(pos.tobytes()).hexdigest() == d["sha"][i]
        opos = O.jittered_grid(H, W, P, s, seed, t).astype("<i4")
        np.testing.assert_array_equal(opos, pos)
        if f"pos_{i}" in d.files:
            np.testing.assert_array_equal(d[f"pos_{i}"], pos)


def test_counter_indexed_philox_stream_pinned_to_numpy():
    """The device generator's model (counter-indexed Philox4x64-10 blocks,
    low/high uint32 halves, Lemire acceptance) reproduces numpy's Generator:
    raw blocks, bounded draws, and whole grids — the golden ones included."""
    for seed, t in [(0, 0), (11, 3), (2 ** 64 - 1, 7), (123456789012345, 2)]:
        raw = np.random.Philox(key=[seed, t]).random_raw(12)
        for b in range(3):
            assert O.philox4x64_10([b + 1, 0, 0, 0], O.philox_key(seed, t)) == \
                [int(v) for v in raw[4 * b:4 * b + 4]]
        g = np.random.Generator(np.random.Philox(key=[seed, t]))
        a = g.integers(0, 4, size=2)
        b_ = g.integers(-2, 3, size=50)
        va, j = O.bounded_draws(seed, t, 0, 2, 4)
        vb, _ = O.bounded_draws(seed, t, j, 50, 5)
        np.testing.assert_array_equal(a, va)
        np.testing.assert_array_equal(b_, vb - 2)
    d = np.load(GOLDEN / "grids.npz")
    for key in d["keys"]:
        H, W, P, s, seed, t = (int(v) for v in key)
        np.testing.assert_array_equal(O.jittered_grid_counter(H, W, P, s, seed, t),
                                      O.jittered_grid(H, W, P, s, seed, t))
