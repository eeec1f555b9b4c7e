"""Offline build_tree against the reference.

GPU: the device KL + local-search build of every reference-built tree we
hold (the synthetic K=200 P=64 / P=100 trees of the benchmark, whose
FEPLLTR1 sha256 the reference wrote into tree_partitions_P*.json, and the
trees of the reference's own restore-test scenarios, stored as FEPLLTR1
bytes) is byte-identical.  CPU: the host parts (level sizes, validation,
seeding + greedy fill, collapse) against the reference's rules.
"""

import hashlib
import json

import numpy as np
import pytest
from conftest import GOLDEN

import fepll_oracle as O  # noqa: F401  (conftest path setup)


def _sha_of_tree(tree, tmp_path, name="t.tr"):
    from paper_1710_08124_b200 import tree_write

    p = tmp_path / name
    tree_write(tree, p)
    return hashlib.sha256(p.read_bytes()).hexdigest(), p.read_bytes()


def test_auto_level_sizes_and_validation():
    from paper_1710_08124_b200 import DataError, auto_level_sizes, build_tree, synthetic

    assert auto_level_sizes(200) == (64, 32, 16, 8, 4, 2, 1)   # pkg/tests/test_tree.py:204-209
    assert auto_level_sizes(1) == ()
    assert auto_level_sizes(5) == (2, 1)
    m = synthetic.synthetic_gmm(8, 16, 0, 0.95)
    for bad in [(8, 1), (4, 4, 1), (4, 2), (2, 4, 1)]:
        with pytest.raises(DataError):
            build_tree(m, bad)


def test_seeding_and_fill_match_reference_rules():
    """With the local search off (sweeps=0) and the divergences given, the
    partition comes from the host seeding + greedy fill alone; compare with
    a direct restatement run on the same matrix."""
    from paper_1710_08124_b200 import balanced_cluster, synthetic

    rng = np.random.default_rng(3)
    X = rng.standard_normal((40, 5))
    D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    comps = [None] * 40
    parts = balanced_cluster(comps, 8, 2, seed=5, sweeps=0, divergences=D)
    sizes = sorted(len(p) for p in parts)
    assert sizes == [5] * 8
    assert sorted(np.concatenate(parts).tolist()) == list(range(40))
    # reference rule: the first medoid is default_rng(seed).integers(n)
    first = int(np.random.default_rng(5).integers(40))
    assert any(first in p for p in parts)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [64, 100])
def test_build_tree_bytes_equal_reference_synthetic(P, tmp_path):
    from paper_1710_08124_b200 import build_tree, synthetic

    meta = json.loads((GOLDEN / f"tree_partitions_P{P}.json").read_text())
    model = synthetic.synthetic_gmm(200, P, 0, 0.95)
    tree = build_tree(model, seed=0)
    sha, _ = _sha_of_tree(tree, tmp_path)
    assert sha == meta["reference_tree_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("name,kw", [("basics", dict(seed=0)), ("estimates16", dict(level_sizes=(2, 1), seed=0)),
                                     ("workers64", dict(seed=0)), ("tree16", dict(seed=0, rho=1.0))])
def test_build_tree_bytes_equal_reference_scenarios(name, kw, tmp_path):
    from paper_1710_08124_b200 import build_tree, model_read

    d = np.load(GOLDEN / f"solver_{name}.npz")
    mp = tmp_path / "m.gm"
    mp.write_bytes(d["model"].tobytes())
    model = model_read(mp)
    tree = build_tree(model, **kw)
    _, data = _sha_of_tree(tree, tmp_path)
    assert data == d["tree"].tobytes()


@pytest.mark.gpu
def test_pairwise_kl_matches_oracle():
    """Device Tr(C_a^-1 C_b) contraction vs the host einsum of tree.py:104."""
    from paper_1710_08124_b200 import pairwise_symmetric_kl, synthetic
    from paper_1710_08124_b200.tree_build import _cov_and_inv

    m = synthetic.synthetic_gmm(30, 64, 1, 0.95)
    kl = pairwise_symmetric_kl(m.components)
    covs = np.stack([_cov_and_inv(c)[0] for c in m.components])
    invs = np.stack([_cov_and_inv(c)[1] for c in m.components])
    t = np.einsum("aij,bji->ab", invs, covs)
    ref = 0.5 * (t + t.T) - 64
    np.fill_diagonal(ref, 0.0)
    np.testing.assert_allclose(kl, ref, rtol=1e-12, atol=1e-9)
    assert np.array_equal(kl, kl.T)
