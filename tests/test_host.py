"""CPU tests of the host side: C-ABI surface, plan packing, model/tree I/O,
sampling plans, operator closed forms, API validation.  No GPU needed."""

import hashlib
import re
from pathlib import Path

import numpy as np
import pytest
from conftest import GOLDEN, ROOT, load_golden

import fepll_oracle as O
from paper_1710_08124_b200 import (DataError, RestorationConfig, beta_schedule, gain_operator,
                                   identity_operator, jitter_rng, jittered_grid, mask_operator,
                                   model_read, model_write, regular_grid, restore, synthetic,
                                   tree_read, tree_write)
from paper_1710_08124_b200 import _native as N
from paper_1710_08124_b200.device_ops import frobenius_norm_sq_ata
from paper_1710_08124_b200.plan import pack_plan, swizzle128_kmajor, tf32_split
from paper_1710_08124_b200.tree import star_tree, tree_partitions, tree_topology


# ---------------------------------------------------------------- C ABI
def header_symbols():
    text = (ROOT / "include" / "fepll_b200.h").read_text()
    return sorted(set(re.findall(r"\b(fepll_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()  # loads libfepll_b200.so (no GPU needed)
    declared = header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) <= set(N.exported_symbols()) | {"fepll_debug_ws_trace"}
    assert lib.fepll_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


# ---------------------------------------------------------------- plan packing
def test_tf32_split_precision():
    rng = np.random.default_rng(0)
    a = (rng.standard_normal(10000) * 10.0 ** rng.uniform(-3, 3, 10000)).astype(np.float32)
    hi, lo = tf32_split(a)
    assert np.all((hi.view(np.uint32) & 0x1FFF) == 0)          # 10-bit mantissa
    lo_t = (lo.view(np.uint32) & 0xFFFFE000).view(np.float32)  # what the MMA reads
    err = np.abs(hi.astype(np.float64) + lo_t - a) / np.abs(a)
    assert err.max() < 2.0 ** -20


def test_swizzle128_is_a_permutation_of_16b_chunks():
    rng = np.random.default_rng(1)
    m = rng.standard_normal((32, 64)).astype(np.float32)
    img = swizzle128_kmajor(m)
    for ka in range(2):
        atom = img[ka * 32 * 32:(ka + 1) * 32 * 32].reshape(32, 8, 4)
        for r in range(32):
            for ch in range(8):
                np.testing.assert_array_equal(atom[r, ch ^ (r % 8)], m[r, ka * 32 + 4 * ch:ka * 32 + 4 * ch + 4])


@pytest.mark.parametrize("P", [64, 100])
def test_pack_plan_layout(P, models):
    model, tree = models[P]
    h = pack_plan(model, tree, [10.0, 20.0])
    topo = h["topo"]
    comps = [n.component for n in tree.bfs_nodes()]
    for u in range(topo.n_nodes):
        nk = topo.child_count[u]
        if nk == 0:
            continue
        kids = topo.child_list[topo.child_start[u]:topo.child_start[u] + nk]
        G = h["grp_basis"][h["grp_off64"][u]:h["grp_off64"][u] + P * h["grp_width"][u]]
        G = G.reshape(P, h["grp_width"][u])
        np.testing.assert_array_equal(G, np.concatenate([comps[v].kept_basis for v in kids], axis=1))
        for v in kids:
            assert h["tc_child_col"][v] % 16 == 0
            c0 = h["tc_w_off"][u] + h["tc_child_col"][v]
            r = comps[v].kept_basis.shape[1]
            np.testing.assert_array_equal(h["tc_w"][:, c0 + r:c0 + (r + 15) // 16 * 16], 0)
        assert h["tc_npad"][u] % 16 == 0


def test_path_costs_reproduce_reference_counters(models):
    """Counters derived from the leaf histogram equal the reference's
    per-patch tree_select counters (tree.py:413-427)."""
    g = load_golden("cfg1")
    model, tree = models[64]
    h = pack_plan(model, tree, [1.0], with_tc=False)
    for t in range(g["labels"].shape[0]):
        hist = np.bincount(g["labels"][t], minlength=200)
        assert int(hist @ h["path_evals"]) == int(g["evals"][t])
        assert int(hist @ h["path_mults"]) == int(g["sel_mults"][t])


def test_star_tree_reproduces_exhaustive_counters(models):
    """No-tree profile (solver.py:154-157): the star tree's path costs give
    K evaluations and P + sum_k score_flat_cost(r_k, P) multiplies per patch,
    the golden notree64 counters."""
    g = load_golden("notree64")
    model, _ = models[64]
    star = star_tree(model)
    topo = tree_topology(star)
    assert topo.n_nodes == 201 and topo.child_count[0] == 200
    np.testing.assert_array_equal(topo.leaf_index[1:], np.arange(200))
    h = pack_plan(model, star, [1.0], with_tc=True)
    assert h["grp_width"][0] == sum(c.kept_basis.shape[1] for c in model.components)
    for t in range(g["labels"].shape[0]):
        hist = np.bincount(g["labels"][t], minlength=200)
        assert int(hist @ h["path_evals"]) == int(g["evals"][t])
        assert int(hist @ h["path_mults"]) == int(g["sel_mults"][t])


# ---------------------------------------------------------------- model / tree I/O
def test_model_roundtrip_bit_exact(tmp_path, models):
    model, _ = models[64]
    p = tmp_path / "m.bin"
    model_write(model, p)
    m2 = model_read(p)
    p2 = tmp_path / "m2.bin"
    model_write(m2, p2)
    assert p.read_bytes() == p2.read_bytes()


def test_tree_roundtrip_and_partitions(tmp_path, models):
    model, tree = models[64]
    p = tmp_path / "t.bin"
    tree_write(tree, p)
    t2 = tree_read(p)
    assert t2.level_sizes == (1, 2, 4, 8, 16, 32, 64, 200)
    assert tree_partitions(t2) == tree_partitions(tree)


@pytest.mark.parametrize("mutate", ["magic", "truncate", "trailing"])
def test_tree_file_corruption_rejected(tmp_path, models, mutate):
    _, tree = models[64]
    p = tmp_path / "t.bin"
    tree_write(tree, p)
    data = p.read_bytes()
    if mutate == "magic":
        data = b"XXXXXXXX" + data[8:]
    elif mutate == "truncate":
        data = data[:-5]
    else:
        data = data + b"\0"
    p.write_bytes(data)
    with pytest.raises(DataError):
        tree_read(p)


# ---------------------------------------------------------------- sampling plans
def test_grid_coverage_and_bounds():
    from paper_1710_08124_b200.patches import axis_anchors

    for (H, W, P, s) in [(64, 64, 64, 6), (41, 53, 64, 3), (37, 29, 100, 4), (33, 47, 64, 1)]:
        side = int(np.sqrt(P))
        base = regular_grid(H, W, P, s).positions
        for seed in range(5):
            g = jittered_grid(H, W, P, s, jitter_rng(seed, 2)).positions
            assert g.shape == base.shape
            assert np.abs(g - base).max() <= (side - s) // 2
            cov = np.zeros((H, W), int)
            for r, c in g:
                cov[r:r + side, c:c + side] += 1
            assert cov.min() >= 1
        assert base.shape[0] == axis_anchors(H, side, s).size * axis_anchors(W, side, s).size


def test_spacing_equal_side_is_regular():
    g = jittered_grid(40, 40, 64, 8, jitter_rng(5, 0))
    np.testing.assert_array_equal(g.positions, regular_grid(40, 40, 64, 8).positions)


# ---------------------------------------------------------------- operators
@pytest.mark.parametrize("name", ["deblur96", "sr96"])
def test_frobenius_closed_form_matches_fft(name):
    from conftest import golden_inputs

    g, A, *_ = golden_inputs(name)
    assert frobenius_norm_sq_ata(A) == pytest.approx(O.frob_ata(O.Op(A)), rel=1e-12)


def test_frobenius_pixel_kinds():
    rng = np.random.default_rng(3)
    m = mask_operator(rng.random((16, 16)) > 0.5)
    gn = gain_operator(rng.random((16, 16)))
    for A in (m, gn, identity_operator((16, 16))):
        assert frobenius_norm_sq_ata(A) == pytest.approx(O.frob_ata(O.Op(A)), rel=1e-14)


# ---------------------------------------------------------------- API validation
def test_beta_schedule_values():
    b = beta_schedule(20.0 / 255.0, 1.0, (1, 4, 8, 16, 32))
    assert abs(b[0] - 162.5625) < 1e-9
    with pytest.raises(DataError):
        beta_schedule(0.0, 1.0, (1,))


def test_config_validation():
    with pytest.raises(DataError):
        RestorationConfig(sigma=20.0, iterations=3).validate()
    with pytest.raises(DataError):
        RestorationConfig(sigma=-1.0).validate()
    with pytest.raises(DataError):
        RestorationConfig(sigma=20.0, sampling="random").validate()


def test_restore_validates_before_touching_the_device(models):
    model, tree = models[64]
    y = np.zeros((32, 32))
    A = identity_operator((32, 32))
    with pytest.raises(DataError, match="tree"):
        restore(y, A, model, None, RestorationConfig(sigma=20.0))
    with pytest.raises(DataError, match="spacing"):
        restore(y, A, model, tree, RestorationConfig(sigma=20.0, spacing=9))
    with pytest.raises(DataError, match="shape"):
        restore(np.zeros((30, 32)), A, model, tree, RestorationConfig(sigma=20.0))
    with pytest.raises(DataError, match="full-rank"):
        restore(y, A, model, tree, RestorationConfig(sigma=20.0, use_flat_tail=False))


# ---------------------------------------------------------------- reference-native objects
REF_SRC = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF_SRC.exists(), reason="the reference package is only in the build container")
def test_reference_objects_pack_like_native_ones():
    """The reference's own GmmModel / GmmTree / DegradationOperator /
    RestorationConfig objects go through the drop-in's host side (duck
    typing): the packed device plan is byte-identical to the one built from
    the package's own types, the closed-form ||A^T A||_F^2 equals the
    reference's, the plan-cache key is computable, and validation raises the
    same errors."""
    import sys

    sys.path.insert(0, str(REF_SRC))
    from fepll import operators as rops
    from fepll.gmm import FlatTailComponent as RComp, GmmModel as RModel
    from fepll.solver import RestorationConfig as RConfig
    from fepll.tree import build_tree as rbuild_tree

    from paper_1710_08124_b200.solver import _plan_key

    model = synthetic.synthetic_gmm(200, 64, 0, 0.95)
    tree = synthetic.baseline_tree(model)
    rmodel = RModel(64, [RComp(c.weight, c.kept_basis, c.kept_eigenvalues, c.tail_value)
                         for c in model.components], model.rho)
    rtree = rbuild_tree(rmodel, seed=0)
    betas = beta_schedule(25.0 / 255.0, 1.0, (1, 4, 8, 16, 32))
    a, b = pack_plan(model, tree, betas), pack_plan(rmodel, rtree, betas)
    for k in ("grp_basis", "node_const", "node_nu_tail", "grp_sqw", "mbasis", "shrink", "gtail",
              "tc_hi", "tc_lo", "tc_x", "tc_w", "path_evals", "path_mults"):
        assert np.array_equal(a[k], b[k]), k
    for A in (rops.identity_operator((64, 64)), rops.mask_operator(np.random.default_rng(0).random((64, 64)) < .5),
              rops.convolution_operator(rops.gaussian_kernel(1.6, 4), (64, 64)),
              rops.decimate_operator(3, (63, 63), rops.gaussian_kernel(1.2, 3))):
        assert frobenius_norm_sq_ata(A) == pytest.approx(rops.frobenius_norm_sq_ata(A), rel=1e-12)
        _plan_key(A, rmodel, rtree, RConfig(sigma=20.0), 1, None, "tensor", None)
    y = np.zeros((64, 64))
    A = rops.identity_operator((64, 64))
    with pytest.raises(DataError, match="tree"):
        restore(y, A, rmodel, None, RConfig(sigma=20.0))
    with pytest.raises(DataError, match="spacing"):
        restore(y, A, rmodel, rtree, RConfig(sigma=20.0, spacing=9))
    with pytest.raises(DataError):
        restore(y, A, rmodel, rtree, RConfig(sigma=20.0, iterations=2))


def test_phase_and_iteration_times_from_timestamp_marks():
    """restore()'s timed CUDA-graph replay hands the phase bookkeeping a list
    of mark names and the milliseconds between consecutive marks
    (Restorer.run_timed_graph): every interval is attributed to the mark that
    closes it, the stretch into an iteration's "start" mark counts as gap,
    and IterationStats.times gets the reference's keys
    (pkg/src/fepll/solver.py:206-254) in seconds."""
    from paper_1710_08124_b200.solver import Restorer

    names = ["start", "init", "start", "extract", "select", "wiener", "aggregate",
             "start", "extract", "select", "wiener", "aggregate", "image_solve"]
    ms = [0.5, 0.01, 1.0, 2.0, 3.0, 4.0, 0.02, 1.5, 2.5, 3.5, 4.5, 5.5]
    timer = {"_marks": [(n, None) for n in names], "_ms": ms}
    ph = Restorer.phase_times(timer)
    assert ph == {"init": 0.5, "gap": 0.01 + 0.02, "extract": 2.5, "select": 4.5, "wiener": 6.5,
                  "aggregate": 8.5, "image_solve": 5.5}
    assert abs(sum(ph.values()) - sum(ms)) < 1e-12
    it = Restorer.iteration_times(timer)
    assert it == [{"grid": 0.0, "extract": 1e-3, "select": 2e-3, "estimate": 3e-3, "reproject": 4e-3},
                  {"grid": 0.0, "extract": 1.5e-3, "select": 2.5e-3, "estimate": 3.5e-3, "reproject": 4.5e-3,
                   "image_solve": 5.5e-3}]
