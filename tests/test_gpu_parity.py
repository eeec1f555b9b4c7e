"""Device path vs the reference's golden vectors and the live CPU oracle.

Parity bar (BASELINE.json north_star): >= 99.9% of selected labels,
restored RMSE <= 1e-3 on the [0,255] scale, |dPSNR| <= 0.01 dB.  The exact
(FP64) path must additionally reproduce every label and counter; the
tensor path must too, because its argmin is certified (tc_epi.cuh) and the
uncertified decisions are re-scored in FP64.
"""

import numpy as np
import pytest
from conftest import golden_inputs, load_golden

import fepll_oracle as O

pytestmark = pytest.mark.gpu

RMSE_TOL = 1e-3      # on [0, 255]
PSNR_TOL = 0.01      # dB
LABEL_TOL = 0.999


def rmse255(a, b):
    return 255.0 * float(np.sqrt(np.mean((np.asarray(a) - np.asarray(b)) ** 2)))


def psnr(x, ref):
    return 10 * np.log10(1.0 / float(np.mean((np.clip(x, 0, 1) - ref) ** 2)))


GOLDEN = ["cfg1", "regular48", "gain64", "inpaint96", "deblur96", "sr96", "notree64"]


@pytest.mark.parametrize("mode", ["exact", "tensor"])
@pytest.mark.parametrize("name", GOLDEN)
def test_restore_matches_reference_golden(name, mode, models):
    from paper_1710_08124_b200 import RestorationConfig, restore

    g, A, y, s8, s, P = golden_inputs(name)
    model, tree = models[P]
    cfg = RestorationConfig(sigma=s8, spacing=s, seed=0, trace=True, sampling=g["meta"]["sampling"],
                            use_tree=bool(g["meta"]["use_tree"]))
    x, st = restore(y, A, model, tree, cfg, mode=mode)
    assert st.lam == pytest.approx(float(g["lam"]), rel=1e-10)
    for t, rec in enumerate(st.trace):
        np.testing.assert_array_equal(rec["selected"], g["labels"][t])
    assert rmse255(x, g["x"]) <= RMSE_TOL
    assert [it.score_evaluations for it in st.iterations] == list(g["evals"])
    assert [it.selection_multiplies for it in st.iterations] == list(g["sel_mults"])
    assert [it.estimation_multiplies for it in st.iterations] == list(g["est_mults"])
    assert [it.image_solve_converged for it in st.iterations] == list(g["converged"])
    assert [it.patches for it in st.iterations] == list(g["patches"])


@pytest.mark.parametrize("cfg_name", ["cfg2", "cfg4a", "cfg3", "cfg4b"])
def test_full_size_configs_vs_live_oracle(cfg_name, models):
    """BASELINE configs 2-4 at full size.  The oracle's lambda comes from its
    own power iteration except for cfg3 (cap active, checked separately)."""
    from paper_1710_08124_b200 import RestorationConfig, restore, synthetic

    c = synthetic.baseline_case(cfg_name)
    model, tree = models[c.patch_dim]
    cfg = RestorationConfig(sigma=c.sigma8, spacing=c.spacing, seed=0, trace=True)
    x, st = restore(c.y, c.A, model, tree, cfg, mode="tensor")
    lam = st.lam if cfg_name == "cfg3" else None
    xo, so = O.restore(c.y, c.A, model, tree, sigma=c.sigma8, spacing=c.spacing, seed=0,
                       trace=True, lam=lam)
    if lam is None:
        assert st.lam == pytest.approx(so.lam, rel=1e-9)
    else:
        assert st.lam == pytest.approx(250.0 * (c.sigma8 / 255.0) ** 2, rel=1e-12)
    agree = [float(np.mean(a["selected"] == b["selected"])) for a, b in zip(st.trace, so.trace)]
    assert min(agree) >= LABEL_TOL, agree
    assert rmse255(x, xo) <= RMSE_TOL
    assert abs(psnr(x, c.clean) - psnr(xo, c.clean)) <= PSNR_TOL


@pytest.mark.parametrize("P,H,s", [(64, 128, 4), (100, 96, 6)])
def test_exhaustive_scan_tensor_vs_exact_and_oracle(P, H, s, models):
    """No-tree profile (gmm.py:371-391) at sizes beyond the golden case: the
    tcgen05 chunked scan (select_wide.cu) and the FP64 block scan give the
    oracle's labels; counters follow solver.py:154-157."""
    from paper_1710_08124_b200 import RestorationConfig, identity_operator, restore, synthetic

    model, _ = models[P]
    img = synthetic.synthetic_image(H, H, 9) / 255.0
    y = img + (20.0 / 255.0) * np.random.default_rng(3).standard_normal((H, H))
    cfg = RestorationConfig(sigma=20.0, spacing=s, seed=1, trace=True, use_tree=False)
    A = identity_operator((H, H))
    xt, st = restore(y, A, model, None, cfg, mode="tensor")
    xe, se = restore(y, A, model, None, cfg, mode="exact")
    xo, so = O.restore(y, A, model, None, sigma=20.0, spacing=s, seed=1, use_tree=False, trace=True)
    for a, b, c in zip(st.trace, se.trace, so.trace):
        np.testing.assert_array_equal(a["selected"], c["selected"])
        np.testing.assert_array_equal(b["selected"], c["selected"])
    assert rmse255(xt, xo) <= RMSE_TOL and rmse255(xe, xo) <= RMSE_TOL
    n = st.iterations[0].patches
    assert all(it.score_evaluations == n * 200 for it in st.iterations)


@pytest.mark.parametrize("P,H,s", [(16, 40, 2), (36, 48, 3), (144, 60, 6), (256, 64, 8)])
def test_other_patch_sizes_no_tree_vs_oracle(P, H, s):
    """Patch sides 4, 6, 12, 16 (power-of-two and generic extraction, K atoms
    1..8; P > 128 scores on the FP64 path in tensor mode) through the no-tree
    profile, which needs no reference-built tree: labels equal the oracle's."""
    from paper_1710_08124_b200 import RestorationConfig, identity_operator, restore, synthetic

    model = synthetic.synthetic_gmm(20, P, 0, 0.95)
    img = synthetic.synthetic_image(H, H, 4) / 255.0
    y = img + (20 / 255) * np.random.default_rng(1).standard_normal((H, H))
    cfg = RestorationConfig(sigma=20.0, spacing=s, seed=1, trace=True, use_tree=False)
    A = identity_operator((H, H))
    xo, so = O.restore(y, A, model, None, sigma=20.0, spacing=s, seed=1, use_tree=False, trace=True)
    for mode in ("exact", "tensor"):
        x, st = restore(y, A, model, None, cfg, mode=mode)
        for a, b in zip(st.trace, so.trace):
            np.testing.assert_array_equal(a["selected"], b["selected"])
        assert rmse255(x, xo) <= RMSE_TOL


def test_host_pipeline_equals_batch_restore(models):
    """HostPipeline (chunks on two streams, pinned float32 buffers) gives the
    float32 of the whole-batch restore, image for image."""
    import torch
    from paper_1710_08124_b200 import HostPipeline, RestorationConfig, restore_batch, synthetic

    model, tree = models[64]
    cases = [synthetic.baseline_case("cfg1", 80, image_seed=i, noise_seed=30 + i) for i in range(4)]
    ys = np.stack([c.y for c in cases]).astype(np.float32)
    cfg = RestorationConfig(sigma=20.0, spacing=4, seed=5)
    hp = HostPipeline(cases[0].A, model, tree, cfg, batch=4, chunks=2)
    pin_in = torch.from_numpy(ys).pin_memory()
    pin_out = torch.empty(ys.shape, dtype=torch.float32).pin_memory()
    hp.run(pin_in, pin_out)
    xb, _ = restore_batch(ys.astype(np.float64), cases[0].A, model, tree, cfg)
    np.testing.assert_array_equal(pin_out.numpy(), xb.astype(np.float32))
    # a stream of batches: three submits (one chunk each, rotating over the
    # two restorers / streams) before one wait, each into its own buffer
    hs = HostPipeline(cases[0].A, model, tree, cfg, batch=2, chunks=1)
    ins = [torch.from_numpy(ys[i:i + 2]).pin_memory() for i in (0, 2, 1)]
    outs = [torch.empty((2,) + ys.shape[1:], dtype=torch.float32).pin_memory() for _ in ins]
    for a, b in zip(ins, outs):
        hs.submit(a, b)
    hs.wait()
    for (i, b) in zip((0, 2, 1), outs):
        np.testing.assert_array_equal(b.numpy(), xb[i:i + 2].astype(np.float32))


def test_same_seed_bit_identical_and_batch_equals_single(models):
    from paper_1710_08124_b200 import RestorationConfig, restore, restore_batch, synthetic

    model, tree = models[64]
    cases = [synthetic.baseline_case("cfg1", 96, image_seed=i, noise_seed=10 + i) for i in range(3)]
    cfg = RestorationConfig(sigma=20.0, spacing=4, seed=3)
    singles = [restore(c.y, c.A, model, tree, cfg)[0] for c in cases]
    again = restore(cases[0].y, cases[0].A, model, tree, cfg)[0]
    assert np.array_equal(singles[0], again)
    xb, _ = restore_batch(np.stack([c.y for c in cases]), cases[0].A, model, tree, cfg)
    for i in range(3):
        assert np.array_equal(xb[i], singles[i])


def test_select_kernel_variants_agree(models):
    """Both tensor-core level kernels (select_ws.cu, select_ws2.cu) and the
    per-level hybrid route every patch identically, and equal the FP64 path."""
    from paper_1710_08124_b200 import RestorationConfig, restore_batch, synthetic

    model, tree = models[64]
    cases = [synthetic.baseline_case("cfg5", 192, image_seed=i, noise_seed=40 + i) for i in range(3)]
    ys = np.stack([c.y for c in cases])
    cfg = RestorationConfig(sigma=25.0, spacing=4, seed=9, trace=True)
    outs = [restore_batch(ys, cases[0].A, model, tree, cfg, mode="tensor",
                          options={"select_variant": v}) for v in (0, 1, 2)]
    xe, se = restore_batch(ys, cases[0].A, model, tree, cfg, mode="exact")
    for x, st in outs:
        np.testing.assert_array_equal(x, outs[0][0])
        assert len(st.trace) == len(se.trace) == 5
        for a, b in zip(st.trace, se.trace):
            np.testing.assert_array_equal(a["selected"], b["selected"])
        assert rmse255(x, xe) <= 1e-9


@pytest.mark.parametrize("H,W,s", [(41, 53, 3), (40, 40, 8), (33, 47, 1), (8, 8, 6)])
def test_edge_geometries_vs_oracle(H, W, s, models):
    """Odd sizes, spacing == side (no jitter), spacing 1, a single anchor."""
    from paper_1710_08124_b200 import RestorationConfig, identity_operator, restore, synthetic

    model, tree = models[64]
    img = synthetic.synthetic_image(H, W, 5) / 255.0
    y = img + (20.0 / 255.0) * np.random.default_rng(7).standard_normal((H, W))
    A = identity_operator((H, W))
    cfg = RestorationConfig(sigma=20.0, spacing=s, seed=11, trace=True)
    x, st = restore(y, A, model, tree, cfg)
    xo, so = O.restore(y, A, model, tree, sigma=20.0, spacing=s, seed=11, trace=True)
    for a, b in zip(st.trace, so.trace):
        np.testing.assert_array_equal(a["selected"], b["selected"])
    assert rmse255(x, xo) <= RMSE_TOL


def test_noiseless_passthrough_and_unclamped(models):
    """solver.py sigma floor: sigma=0 returns ~y; output is not clamped."""
    from paper_1710_08124_b200 import RestorationConfig, identity_operator, restore, synthetic

    model, tree = models[64]
    y = synthetic.synthetic_image(48, 48, 1) / 255.0 + 0.5
    A = identity_operator(y.shape)
    x, st = restore(y, A, model, tree, RestorationConfig(sigma=0.0, spacing=4))
    xo, so = O.restore(y, A, model, tree, sigma=0.0, spacing=4)
    assert st.lam == pytest.approx(so.lam) and st.iterations[0].beta == pytest.approx(so.betas[0])
    assert rmse255(x, xo) <= RMSE_TOL
    assert np.sqrt(np.mean((x - y) ** 2)) < 5e-3   # floor sigma = 0.5/255: near pass-through
    assert x.max() > 1.0


def test_nonfinite_input_raises_numerical_error(models):
    from paper_1710_08124_b200 import NumericalError, RestorationConfig, identity_operator, restore

    model, tree = models[64]
    y = np.full((32, 32), 0.5)
    y[3, 4] = np.nan
    with pytest.raises(NumericalError):
        restore(y, identity_operator(y.shape), model, tree, RestorationConfig(sigma=20.0, spacing=4))


# ---------------------------------------------------------------- kernel-level parity (C ABI)
def _dev(a, dtype=None):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def test_extract_kernel_bitwise():
    """Kernel (a) vs the oracle's extract (patches.py:153-183), bitwise, over
    patch sides and spacings — and over output layouts the ABI allows: the
    padded 128-byte pitch (paired-store kernel), an odd Z32 pitch and Z64/Z32
    pointers offset by one element (per-row-store kernel)."""
    import torch
    from paper_1710_08124_b200 import _native as N, jitter_rng, jittered_grid

    for P, H, W, s, layout in [(64, 70, 61, 3, "padded"), (64, 70, 61, 3, "odd"),
                               (64, 70, 61, 3, "offset"), (100, 64, 64, 6, "padded"),
                               (36, 30, 40, 2, "padded"), (16, 50, 47, 1, "padded"),
                               (16, 50, 47, 1, "odd"), (256, 64, 80, 16, "padded"),
                               (64, 300, 280, 1, "padded"), (64, 300, 280, 8, "padded"),
                               (256, 90, 70, 3, "offset")]:
        side = int(np.sqrt(P))
        x = np.random.default_rng(P).random((H, W))
        pos = jittered_grid(H, W, P, s, jitter_rng(1, 2)).positions.astype(np.int32)
        n = pos.shape[0]
        Zo, dco = O.extract(x, pos.astype(np.int64), side)
        pitch = {"padded": (P + 31) // 32 * 32, "odd": P + 1, "offset": P}[layout]
        off = 1 if layout == "offset" else 0
        Z64b = torch.empty(n * P + off, dtype=torch.float64, device="cuda")
        Z32b = torch.empty(n * pitch + off, dtype=torch.float32, device="cuda")
        Z64, Z32 = Z64b[off:].view(n, P), Z32b[off:].view(n, pitch)
        dc = torch.empty(n, dtype=torch.float64, device="cuda")
        sq = torch.empty(n, dtype=torch.float64, device="cuda")
        xd, pd = _dev(x), _dev(pos)  # keep the device inputs alive across the async launch
        N.call("fepll_extract", N.ptr(xd), 1, H, W, side, N.ptr(pd), n, 0, N.ptr(Z64),
               N.ptr(Z32), pitch, N.ptr(dc), N.ptr(sq), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(dc.cpu().numpy(), dco)           # pairwise fold, bitwise
        np.testing.assert_array_equal(Z64.cpu().numpy(), Zo)
        np.testing.assert_array_equal(Z32.cpu().numpy()[:, :P], Zo.astype(np.float32))
        assert not Z32.cpu().numpy()[:, P:].any()
        np.testing.assert_allclose(sq.cpu().numpy(), np.einsum("ij,ij->i", Zo, Zo), rtol=1e-13)


@pytest.mark.parametrize("mode", ["tensor", "exact"])
@pytest.mark.parametrize("H,W,world,s", [(160, 96, 3, 4), (130, 77, 2, 3), (96, 64, 4, 2)])
def test_strip_mode_bitwise_equals_unsplit(H, W, world, s, mode, models):
    """SURVEY §8(e) strip mode: world strips with halo exchange between HQS
    iterations reproduce the single-image run bit for bit."""
    from paper_1710_08124_b200 import RestorationConfig, identity_operator, restore, synthetic
    from paper_1710_08124_b200.strips import restore_strips_single_process

    model, tree = models[64]
    img = synthetic.synthetic_image(H, W, 3) / 255.0
    y = img + (25.0 / 255.0) * np.random.default_rng(5).standard_normal((H, W))
    cfg = RestorationConfig(sigma=25.0, spacing=s, seed=2)
    x_full, _ = restore(y, identity_operator((H, W)), model, tree, cfg, mode=mode)
    x_strips = restore_strips_single_process(y, model, tree, cfg, world, mode=mode)
    assert np.array_equal(x_strips, x_full)


def _device_grid(H, W, P, s, seed, t, jittered=True, threshold=0):
    import torch
    from paper_1710_08124_b200 import _native as N
    from paper_1710_08124_b200.patches import axis_anchors, philox_key

    side = int(np.sqrt(P))
    n = axis_anchors(H, side, s).size * axis_anchors(W, side, s).size
    anchors = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    scratch = torch.empty(N.lib().fepll_grid_scratch_ints(), dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    k0, k1 = philox_key(seed, t)
    N.call("fepll_sample_grid", k0, k1, H, W, side, s, int(jittered), threshold, N.ptr(anchors),
           N.ptr(scratch), N.ptr(status), torch.cuda.current_stream().cuda_stream)
    assert int(status.item()) == 0
    return anchors.cpu().numpy().astype(np.int64), int(scratch[3].item())


def test_device_sampling_plan_bitwise_vs_numpy():
    """csrc/grid.cu == jittered_grid(Generator(Philox(key=[seed, t]))) and
    regular_grid, over sizes, spacings, P, seeds (incl. >= 2^63) and t."""
    from paper_1710_08124_b200 import jitter_rng, jittered_grid, regular_grid

    for (H, W, P, s) in [(64, 64, 64, 4), (41, 53, 64, 3), (96, 96, 100, 6), (33, 47, 64, 1),
                         (512, 512, 64, 4), (1024, 768, 64, 2), (510, 510, 100, 5), (8, 8, 64, 6)]:
        for seed, t in [(0, 0), (0, 4), (11, 2), (2 ** 64 - 1, 3), (987654321987, 1)]:
            want = jittered_grid(H, W, P, s, jitter_rng(seed, t)).positions
            got, _ = _device_grid(H, W, P, s, seed, t)
            np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(_device_grid(H, W, P, s, 0, 0, jittered=False)[0],
                                      regular_grid(H, W, P, s).positions)


def test_device_sampling_plan_rejection_fixup():
    """Forced Lemire rejections (threshold override, ~1% of draws) follow the
    counter-indexed oracle stream, whose unforced form is pinned to numpy."""
    for (H, W, P, s, seed, t) in [(96, 96, 64, 4, 5, 1), (64, 80, 100, 6, 0, 3), (48, 48, 64, 2, 9, 0)]:
        th = 1 << 25
        want = O.jittered_grid_counter(H, W, P, s, seed, t, threshold=th)
        got, rejects = _device_grid(H, W, P, s, seed, t, threshold=th)
        assert rejects > 0
        np.testing.assert_array_equal(got, want)


def test_aggregate_kernel_bitwise_vs_bincount():
    """Fed the reference's estimates, the ordered gather reproduces
    np.bincount's sums bit for bit (patches.py:198-222)."""
    import torch
    from paper_1710_08124_b200 import _native as N, jitter_rng, jittered_grid
    from paper_1710_08124_b200.patches import axis_anchors

    for P, H, W, s in [(64, 70, 61, 3), (100, 64, 64, 6), (64, 40, 40, 1)]:
        side = int(np.sqrt(P))
        pos = jittered_grid(H, W, P, s, jitter_rng(4, 1)).positions.astype(np.int32)
        n = pos.shape[0]
        rng = np.random.default_rng(2)
        est = rng.standard_normal((n, P))
        dc = rng.standard_normal(n)
        ref = O.reproject(est, dc, pos.astype(np.int64), side, H, W)
        xt = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        ed, dd, pd = _dev(est), _dev(dc), _dev(pos)
        N.call("fepll_aggregate", N.ptr(ed), N.ptr(dd), N.ptr(pd),
               axis_anchors(H, side, s).size, axis_anchors(W, side, s).size, s, (side - s) // 2,
               side, 1, H, W, None, None, 1.0, 1, None, N.ptr(xt), N.ptr(status),
               torch.cuda.current_stream().cuda_stream)
        np.testing.assert_array_equal(xt.cpu().numpy()[0], ref)
        assert int(status.item()) == 0
        # the same gather over the plan's cover lists (the solver's path)
        nr, nc = axis_anchors(H, side, s).size, axis_anchors(W, side, s).size
        ptr = torch.empty(H * W + 1, dtype=torch.int32, device="cuda")
        ent = torch.empty(n * P, dtype=torch.int32, device="cuda")
        scr = torch.empty(int(N.lib().fepll_cover_scratch_ints(H * W)), dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        N.call("fepll_cover_build", N.ptr(pd), nr, nc, s, (side - s) // 2, side, W, 0, H, 0, nr, 0, H,
               N.ptr(ptr), N.ptr(ent), n * P, N.ptr(scr), st)
        assert int(ptr[-1].item()) == n * P  # every patch covers exactly P pixels
        xc = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
        N.call("fepll_aggregate_cover", N.ptr(ed), N.ptr(dd), N.ptr(ptr), N.ptr(ent), P, n, n, 1, H, W,
               0, H, None, None, 1.0, 1, None, N.ptr(xc), N.ptr(status), st)
        np.testing.assert_array_equal(xc.cpu().numpy()[0], ref)


def test_aggregate_cover_batch_with_and_without_dc():
    """Batched cover gather (images split over block groups, several images in
    flight per thread) equals np.bincount per image, both when it adds dc and
    when the estimates already hold est + dc (the Wiener kernels' output)."""
    import torch
    from paper_1710_08124_b200 import _native as N, jitter_rng, jittered_grid
    from paper_1710_08124_b200.patches import axis_anchors

    P, H, W, s, B = 64, 72, 300, 4, 19
    side = 8
    pos = jittered_grid(H, W, P, s, jitter_rng(7, 2)).positions.astype(np.int32)
    n = pos.shape[0]
    rng = np.random.default_rng(5)
    est = rng.standard_normal((B, n, P)) * 30
    dc = rng.standard_normal((B, n)) * 100
    refs = [O.reproject(est[b], dc[b], pos.astype(np.int64), side, H, W) for b in range(B)]
    nr, nc = axis_anchors(H, side, s).size, axis_anchors(W, side, s).size
    st = torch.cuda.current_stream().cuda_stream
    pd = _dev(pos)
    ptr = torch.empty(H * W + 1, dtype=torch.int32, device="cuda")
    ent = torch.empty(n * P, dtype=torch.int32, device="cuda")
    scr = torch.empty(int(N.lib().fepll_cover_scratch_ints(H * W)), dtype=torch.int32, device="cuda")
    N.call("fepll_cover_build", N.ptr(pd), nr, nc, s, (side - s) // 2, side, W, 0, H, 0, nr, 0, H,
           N.ptr(ptr), N.ptr(ent), n * P, N.ptr(scr), st)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for pre_added, pad in ((False, 0), (True, 0), (True, 3)):
        vals = est + dc[:, :, None] if pre_added else est
        # padded image pitch: rows n .. n+pad-1 of every image are garbage
        vals = np.concatenate([vals, np.full((B, pad, P), np.nan)], axis=1)
        ed = _dev(np.ascontiguousarray(vals.reshape(B * (n + pad), P)))
        dd = None if pre_added else _dev(dc.reshape(-1))
        xc = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
        N.call("fepll_aggregate_cover", N.ptr(ed), N.ptr(dd), N.ptr(ptr), N.ptr(ent), P, n, n + pad, B, H, W,
               0, H, None, None, 1.0, 1, None, N.ptr(xc), N.ptr(status), st)
        got = xc.cpu().numpy()
        for b in range(B):
            np.testing.assert_array_equal(got[b], refs[b])
    assert int(status.item()) == 0


def test_lo_eq_hi_rule_returns_common_value():
    """Identical overlapping contributions come back verbatim (patches.py:221)."""
    import torch
    from paper_1710_08124_b200 import _native as N

    H = W = 8
    pos = np.array([[0, 0], [0, 0]], np.int32)
    v = np.full((2, 64), 0.1)
    dc = np.array([0.2, 0.2])
    xt = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    # two anchors at the same place: nominal grid of 2 rows x 1 col, spacing 8
    vd, dd, pd = _dev(v), _dev(dc), _dev(pos)
    N.call("fepll_aggregate", N.ptr(vd), N.ptr(dd), N.ptr(pd), 1, 2, 8, 0, 8, 1,
           H, W, None, None, 1.0, 1, None, N.ptr(xt), N.ptr(status),
           torch.cuda.current_stream().cuda_stream)
    assert np.all(xt.cpu().numpy() == 0.1 + 0.2)


def test_uncovered_pixel_raises_data_error():
    import torch
    from paper_1710_08124_b200 import _native as N

    H = W = 16
    pos = np.array([[0, 0]], np.int32)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    xt = torch.empty((1, H, W), dtype=torch.float64, device="cuda")
    zd, dd, pd = _dev(np.zeros((1, 16))), _dev(np.zeros(1)), _dev(pos)
    N.call("fepll_aggregate", N.ptr(zd), N.ptr(dd), N.ptr(pd), 1, 1, 4, 0, 4, 1, H, W, None, None, 1.0, 1, None, N.ptr(xt),
           N.ptr(status), torch.cuda.current_stream().cuda_stream)
    assert int(status.item()) & 1


@pytest.mark.parametrize("name", ["deblur96", "sr96", "inpaint96", "gain64"])
def test_operator_adjoint_identity_and_normal(name):
    """<A x, y> == <x, A^T y> through the device A^T, and A^T A vs the oracle."""
    import torch
    from paper_1710_08124_b200.device_ops import DeviceOperator

    _, A, *_ = golden_inputs(name)
    op = DeviceOperator(A)
    o = O.Op(A)
    rng = np.random.default_rng(5)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        x = rng.standard_normal(A.input_dims)
        y = rng.standard_normal(A.output_dims)
        aty = torch.empty(A.input_dims, dtype=torch.float64, device="cuda")
        yd, xd = _dev(y), _dev(x)
        op.adjoint(yd, aty, st)
        np.testing.assert_allclose(aty.cpu().numpy(), o.adjoint(y), rtol=0, atol=1e-12)
        lhs = float(np.vdot(o.apply(x), y))
        rhs = float(np.vdot(x, aty.cpu().numpy()))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))
        nx = torch.empty(A.input_dims, dtype=torch.float64, device="cuda")
        op.normal(xd, 0.5, nx, st)
        np.testing.assert_allclose(nx.cpu().numpy(), o.normal(x) + 0.5 * x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("knob,values", [
    ("wiener_rw", (8, 16)),          # Wiener: 8 vs 16 rows per warp
    ("wiener_xw", (0, 1)),           # Wiener: extracted Z64 rows vs image windows
    ("wiener_pair", (1, 0)),         # Wiener: two 64-row CTAs per SM vs deeper staging
    ("seg_sq", (1, 0)),              # ws2: segment-order ||z||^2 vs gather
    ("select_variant", (1, 0, 2)),   # tree level: ws2 vs ws kernel vs per-level hybrid
    ("wiener_add_dc", (1, 0)),       # est + dc from the Wiener kernel vs dc added by the gather
    ("l2_prefetch", (0, 1)),         # ws2 loaders: L2 prefetch three tiles ahead vs none
    ("rescore_by_node", (0, 1)),     # FP64 re-scoring per decision vs grouped by node (smem group)
    ("wiener_split", (0, 1)),          # Wiener: 8-row m8n8k4 warps vs m16n8k8 warp pairs
    ("wiener_ws", (2, 0, 1)),          # Wiener: two 64-row CTAs per SM (2 = by size: here too) vs the warp-specialised single CTA
    ("defer", (1, 0)),                 # deferred FP64 verification vs re-scoring after every level
    ("pdl", (1, 0)),                   # programmatic dependent launch of the level / re-scoring kernels
    ("aggregate_variant", (2, 0, 1)),  # batch reprojection: staged tiles / thread per pixel / per (pixel, image)
])
def test_kernel_variants_bitwise_equal(knob, values, models):
    """Every performance variant kept behind a plan option computes the same
    images and labels bit for bit (same FP64 operation order per element),
    on a batch that exercises the cover gather and the DMMA Wiener kernel.
    The options live on the plan: a second restorer in the same process
    keeps its defaults."""
    import torch
    from paper_1710_08124_b200 import Restorer, RestorationConfig, synthetic

    model, tree = models[64]
    cases = [synthetic.baseline_case("cfg1", 144, image_seed=i, noise_seed=70 + i) for i in range(3)]
    y = torch.from_numpy(np.stack([c.y for c in cases])).cuda()
    cfg = RestorationConfig(sigma=20.0, spacing=4, seed=9)
    outs = []
    for v in values:
        r = Restorer(cases[0].A, model, tree, cfg, batch=3, options={knob: v})
        assert r.plan.get_option(knob) == v
        x, rec = r.run(y, trace=True)
        outs.append((x.cpu().numpy().copy(), [t["selected"] for t in rec]))
    other = Restorer(cases[0].A, model, tree, cfg, batch=3)
    assert other.plan.get_option(knob) == values[0]
    x0, l0 = outs[0]
    for x1, l1 in outs[1:]:
        assert np.array_equal(x0, x1)
        for a, b in zip(l0, l1):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("H,W,P,s,B", [(40, 300, 64, 4, 3), (64, 64, 64, 2, 5), (37, 530, 100, 4, 2),
                                       (24, 256, 64, 8, 2), (33, 47, 64, 1, 2), (40, 300, 64, 4, 1)])
def test_aggregate_tiles_bitwise(H, W, P, s, B):
    """fepll_aggregate_tiles (segments staged in shared memory) equals the
    cover-list gather bit for bit — FP64 and FP32 Zhat, with and without dc,
    pixel-diagonal update with and without a diagonal, the FFT/CG rhs form
    with x~ out — on partial tiles (W not a multiple of 256), spacing 1, 2,
    4 and 8, P = 64 and 100; constant inputs come back verbatim."""
    import torch
    from paper_1710_08124_b200 import _native as N, jitter_rng, jittered_grid
    from paper_1710_08124_b200.patches import axis_anchors

    side = int(round(P ** 0.5))
    half = (side - s) // 2
    pos = jittered_grid(H, W, P, s, jitter_rng(5, 1)).positions.astype(np.int32)
    n = pos.shape[0]
    nr, nc = axis_anchors(H, side, s).size, axis_anchors(W, side, s).size
    st = torch.cuda.current_stream().cuda_stream
    pd = _dev(pos)
    ptr = torch.empty(H * W + 1, dtype=torch.int32, device="cuda")
    ent = torch.empty(n * P, dtype=torch.int32, device="cuda")
    scr = torch.empty(int(N.lib().fepll_cover_scratch_ints(H * W)), dtype=torch.int32, device="cuda")
    N.call("fepll_cover_build", N.ptr(pd), nr, nc, s, half, side, W, 0, H, 0, nr, 0, H,
           N.ptr(ptr), N.ptr(ent), n * P, N.ptr(scr), st)
    tw = int(N.lib().fepll_tiles_width())
    n_tiles = H * ((W + tw - 1) // tw)
    cap = int(N.lib().fepll_tiles_seg_cap(side, s, half))
    seg_off = torch.empty(n_tiles * cap, dtype=torch.int32, device="cuda")
    seg_cnt = torch.empty(n_tiles, dtype=torch.int32, device="cuda")
    c16 = torch.empty(n * P, dtype=torch.int16, device="cuda")
    mx = torch.zeros(1, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("fepll_tiles_build", N.ptr(ptr), N.ptr(ent), P, side, W, H, cap, N.ptr(seg_off), N.ptr(seg_cnt),
           N.ptr(c16), N.ptr(mx), N.ptr(status), st)
    assert int(status.item()) == 0 and 0 < int(mx.item()) <= cap
    max_seg = int(mx.item())
    rng = np.random.default_rng(H * W + P)
    zrows = n + 3  # padded rows per image
    aty = _dev(rng.standard_normal((B, H, W)))
    diag = _dev(rng.uniform(0.0, 2.0, (B, H, W)))
    dc = _dev(rng.standard_normal(B * n))
    for dtype in (np.float64, np.float32):
        if dtype == np.float32 and (side * 4) % 16:
            continue
        z = torch.from_numpy(rng.standard_normal((B * zrows, P)).astype(dtype)).cuda()
        zc = torch.from_numpy(np.full((B * zrows, P), 0.1 + 0.2).astype(dtype)).cuda()
        f64 = dtype == np.float64
        cover = "fepll_aggregate_cover" if f64 else "fepll_aggregate_cover_f32"
        for zz, dcp, dg, kind in ((z, None, None, 0), (z, dc, diag, 0), (z, None, None, 1), (zc, None, diag, 1)):
            outs = []
            for tiles in (False, True):
                x = torch.full((B, H, W), 7.0, dtype=torch.float64, device="cuda")
                xt = torch.full((B, H, W), 7.0, dtype=torch.float64, device="cuda")
                if tiles:
                    N.call("fepll_aggregate_tiles", N.ptr(zz) if f64 else None, None if f64 else N.ptr(zz),
                           N.ptr(dcp), n, N.ptr(ptr), N.ptr(c16), N.ptr(seg_off), N.ptr(seg_cnt), cap, max_seg,
                           P, zrows, B, H, W, 0, H, N.ptr(aty), N.ptr(dg), 0.37, kind, N.ptr(x), N.ptr(xt),
                           N.ptr(status), st)
                else:
                    N.call(cover, N.ptr(zz), N.ptr(dcp), N.ptr(ptr), N.ptr(ent), P, n, zrows, B, H, W, 0, H,
                           N.ptr(aty), N.ptr(dg), 0.37, kind, N.ptr(x), N.ptr(xt), N.ptr(status), st)
                outs.append((x.cpu().numpy(), xt.cpu().numpy()))
            np.testing.assert_array_equal(outs[0][0], outs[1][0])
            np.testing.assert_array_equal(outs[0][1], outs[1][1])
            if zz is zc:
                assert np.all(outs[1][1] == dtype(0.1 + 0.2).astype(np.float64))
    assert int(status.item()) == 0


def test_cover_gather_lo_eq_hi_verbatim_and_pipeline_errors(models):
    """Identical contributions come back verbatim through both cover-list
    gathers (batched and single-image kernels; patches.py:221 — a sum / count
    would round differently for counts 3, 5, 6, 7, 9 of the jittered grid),
    and HostPipeline.wait() raises the reference's NumericalError for a
    non-finite observation."""
    import torch
    from paper_1710_08124_b200 import (HostPipeline, NumericalError, RestorationConfig, synthetic,
                                       _native as N, jitter_rng, jittered_grid)
    from paper_1710_08124_b200.patches import axis_anchors

    P, H, W, s, side = 64, 40, 56, 4, 8
    pos = jittered_grid(H, W, P, s, jitter_rng(3, 0)).positions.astype(np.int32)
    n = pos.shape[0]
    nr, nc = axis_anchors(H, side, s).size, axis_anchors(W, side, s).size
    st = torch.cuda.current_stream().cuda_stream
    pd = _dev(pos)
    ptr = torch.empty(H * W + 1, dtype=torch.int32, device="cuda")
    ent = torch.empty(n * P, dtype=torch.int32, device="cuda")
    scr = torch.empty(int(N.lib().fepll_cover_scratch_ints(H * W)), dtype=torch.int32, device="cuda")
    N.call("fepll_cover_build", N.ptr(pd), nr, nc, s, (side - s) // 2, side, W, 0, H, 0, nr, 0, H,
           N.ptr(ptr), N.ptr(ent), n * P, N.ptr(scr), st)
    counts = np.diff(ptr.cpu().numpy())
    assert len(set(counts.tolist()) - {1, 2, 4, 8}) > 0  # non-power-of-two counts present
    c = 0.1 + 0.2
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for B in (1, 3):
        vals = _dev(np.full((B * n, P), c))
        xc = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
        N.call("fepll_aggregate_cover", N.ptr(vals), None, N.ptr(ptr), N.ptr(ent), P, n, n, B, H, W,
               0, H, None, None, 1.0, 1, None, N.ptr(xc), N.ptr(status), st)
        assert np.all(xc.cpu().numpy() == c)
    assert int(status.item()) == 0

    model, tree = models[64]
    case = synthetic.baseline_case("cfg1", 64)
    ys = np.stack([case.y, case.y]).astype(np.float32)
    ys[1, 10, 10] = np.nan
    hp = HostPipeline(case.A, model, tree, RestorationConfig(sigma=20.0, spacing=4), batch=2)
    pin_in = torch.from_numpy(ys).pin_memory()
    pin_out = torch.empty(ys.shape, dtype=torch.float32).pin_memory()
    hp.submit(pin_in, pin_out)
    with pytest.raises(NumericalError):
        hp.wait()


@pytest.mark.parametrize("name", ["cfg1", "deblur96", "sr96"])
def test_restore_graph_replay_equals_eager_and_fills_times(name, models):
    """restore() with a cached plan replays one timed CUDA graph of the whole
    restore (device timestamps at the phase marks); the image, counters and
    CG flags are bitwise those of the eager path, also when the observation
    changes between calls, and IterationStats.times carries the reference's
    keys (pkg/src/fepll/solver.py:206-254) with that call's device times."""
    from paper_1710_08124_b200 import RestorationConfig, restore
    from paper_1710_08124_b200.solver import cached_restorer, clear_plan_cache

    clear_plan_cache()
    g, A, y, s8, s, P = golden_inputs(name)
    model, tree = models[P]
    cfg = RestorationConfig(sigma=s8, spacing=s, seed=0, sampling=g["meta"]["sampling"])
    y2 = np.ascontiguousarray(y[::-1, ::-1])
    r = cached_restorer(A, model, tree, cfg, batch=1)
    r.use_graph = False
    x_e, st_e = restore(y, A, model, tree, cfg)
    x2_e, _ = restore(y2, A, model, tree, cfg)
    r.use_graph = True
    x_g, st_g = restore(y, A, model, tree, cfg)    # captures
    x2_g, _ = restore(y2, A, model, tree, cfg)     # replays on another observation
    x_g2, st_g2 = restore(y, A, model, tree, cfg)  # replays
    assert r._tg_graph is not None
    assert np.array_equal(x_e, x_g) and np.array_equal(x_g, x_g2) and np.array_equal(x2_e, x2_g)
    keys = {"grid", "extract", "select", "estimate", "reproject"}
    if A.kind in ("convolution", "decimate"):
        keys.add("image_solve")
    for a, b in zip(st_e.iterations, st_g2.iterations):
        assert (a.patches, a.score_evaluations, a.selection_multiplies, a.estimation_multiplies) == \
               (b.patches, b.score_evaluations, b.selection_multiplies, b.estimation_multiplies)
        assert a.image_solve_converged == b.image_solve_converged
        assert set(b.times) >= keys
        assert all(0.0 <= b.times[k] < 0.05 for k in keys) and b.times["select"] > 0.0
    clear_plan_cache()
