"""The restoration entry point: drop-in for ``fepll.solver.restore``.

``restore(y, A, model, tree=None, config=None) -> (x, SolverStats)`` keeps
the reference signature, validation and error behaviour
(`pkg/src/fepll/solver.py:161-274`) and accepts the reference's own
``RestorationConfig``/``DegradationOperator``/``GmmModel``/``GmmTree``
objects (duck typing).  The loop body runs on the GPU through the C ABI:

    grid plan -> (a) extract -> (b) select -> (c) Wiener -> (d) aggregate
    -> (e) image update

with all per-iteration state resident in HBM; the host only sequences
launches.  :func:`restore_batch` restores a stack of images that share the
operator and noise level in one pass (the batch of BASELINE config 5).
"""

from __future__ import annotations

import hashlib
import math
import time
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import DataError, DeviceError, NumericalError
from .gmm import score_flat_cost, wiener_flat_cost
from .operators import CgConfig
from .patches import SampleGrid, axis_anchors, jitter_rng, jittered_grid, philox_key, regular_grid
from .device_ops import DeviceOperator
from .plan import DevicePlan
from .tree import star_tree

__all__ = ["RestorationConfig", "IterationStats", "SolverStats", "beta_schedule",
           "restore", "restore_batch", "Restorer", "HostPipeline", "cached_restorer",
           "clear_plan_cache", "SIGMA_FLOOR_8BIT"]

SIGMA_FLOOR_8BIT = 0.5


@dataclass
class RestorationConfig:
    """Same fields and defaults as `pkg/src/fepll/solver.py:63-88`."""

    sigma: float
    iterations: int = 5
    beta_multipliers: tuple = (1.0, 4.0, 8.0, 16.0, 32.0)
    spacing: int = 6
    sampling: str = "jittered"
    use_tree: bool = True
    use_flat_tail: bool = True
    rho: float = 0.95
    seed: int = 0
    cg: CgConfig = field(default_factory=CgConfig)
    workers: int = 1
    trace: bool = False

    def validate(self) -> None:
        _validate_config(self)


def _validate_config(c) -> None:
    if c.sigma < 0:
        raise DataError("sigma must be nonnegative")
    if c.iterations != len(c.beta_multipliers):
        raise DataError(f"iterations {c.iterations} != number of beta multipliers "
                        f"{len(c.beta_multipliers)}")
    if c.sampling not in ("jittered", "regular"):
        raise DataError(f"unknown sampling mode {c.sampling!r}")
    if c.workers < 1:
        raise DataError("workers must be >= 1")
    if c.cg.tolerance <= 0:
        raise DataError("CG tolerance must be positive")
    if c.cg.max_iterations < 1:
        raise DataError("CG needs at least one iteration")


@dataclass
class IterationStats:
    beta: float
    patches: int = 0
    score_evaluations: int = 0
    selection_multiplies: int = 0
    estimation_multiplies: int = 0
    times: dict = field(default_factory=dict)
    image_solve_converged: bool = True
    image_solve_residual: float = 0.0


@dataclass
class SolverStats:
    iterations: list = field(default_factory=list)
    init_seconds: float = 0.0
    total_seconds: float = 0.0
    lam: float = 0.0
    trace: list = field(default_factory=list)
    rescored: list = field(default_factory=list)   # FP64 re-scored decisions / iteration
    repaired: list = field(default_factory=list)   # patches re-descended by the deferred verification

    @property
    def total_patches(self) -> int:
        return sum(it.patches for it in self.iterations)

    @property
    def total_score_evaluations(self) -> int:
        return sum(it.score_evaluations for it in self.iterations)

    @property
    def total_selection_multiplies(self) -> int:
        return sum(it.selection_multiplies for it in self.iterations)

    @property
    def total_estimation_multiplies(self) -> int:
        return sum(it.estimation_multiplies for it in self.iterations)

    def step_seconds(self) -> dict:
        out: dict = {}
        for it in self.iterations:
            for k, v in it.times.items():
                out[k] = out.get(k, 0.0) + v
        return out


def beta_schedule(sigma: float, lam: float, multipliers: Sequence[float]) -> np.ndarray:
    """beta_t = mult_t * lambda / sigma^2 (`pkg/src/fepll/solver.py:135-140`)."""
    if sigma <= 0:
        raise DataError("sigma must be positive (apply the floor first)")
    return np.asarray(multipliers, dtype=np.float64) * lam / (sigma * sigma)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.DeviceError("no CUDA device: the FEPLL loop runs only on the GPU")
    return torch


class Restorer:
    """Reusable device state for one (model, tree, operator, config).

    Plans (packed bases, scratch) are built once; :meth:`run` executes the
    loop for a device-resident batch of observations.
    """

    MODES = {"exact": 0, "tensor": 1}

    def __init__(self, A, model, tree, config, batch: int = 1, lam: float | None = None,
                 mode: str = "tensor", device=None, guard: float = 0.0, strip=None,
                 options: dict | None = None, precision: str = "fp64"):
        _validate_config(config)
        # precision: "fp64" (default) keeps the patch rows and the Wiener
        # estimates in FP64 (bitwise-reproducible, labels identical to the
        # FP64 reference); "fp32-state" stores them in FP32 (no Z64 rows,
        # FP32 est + dc) with FP64 arithmetic throughout and the exact FP64
        # re-scoring from the FP64 image — about half the HBM bytes of
        # extraction, Wiener and reprojection (FP32 state
        # gave no label flips and RMSE ~4e-6 in emulation)
        if precision not in ("fp64", "fp32-state"):
            raise DataError(f"unknown precision {precision!r} (fp64 | fp32-state)")
        self.precision = precision
        # strip mode (strips.StripSpec): A covers the strip's slab of a larger
        # image; only the owned rows are aggregated (denoise, batch 1)
        self.strip = strip
        if strip is not None:
            if A.kind != "identity" or int(batch) != 1:
                raise DataError("strip mode restores one denoising image (identity operator, batch 1)")
            if tuple(A.input_dims) != (strip.slab_hi - strip.slab_lo, strip.W):
                raise DataError("strip operator dims differ from the strip's slab")
        self.config = config
        self.A = A
        self.model = model
        self.tree = tree
        self.batch = int(batch)
        P = int(model.patch_dim)
        side = math.isqrt(P)
        if side * side != P:
            raise DataError(f"model patch_dim {P} is not a perfect square")
        if not 1 <= config.spacing <= side:
            raise DataError(f"spacing must lie in [1, {side}]")
        if config.use_tree:
            if tree is None:
                raise DataError("use_tree requires a search tree")
            if tree.n_leaves != len(model.components):
                raise DataError(f"tree has {tree.n_leaves} leaves but the model has "
                                f"{len(model.components)} components")
        else:
            # exhaustive scan (solver.py:154-157) == descent of the one-level star tree
            tree = self.tree = star_tree(model)
        if not config.use_flat_tail and not bool(np.all(
                [c.kept_basis.shape[1] == P for c in model.components])):
            raise DataError("flat tail disabled: a full-rank model is required")
        A.solve_strategy  # validates the kind
        if mode not in self.MODES:
            raise DataError(f"unknown mode {mode!r} (exact | tensor)")
        torch = _torch()
        self.torch = torch
        self.device = torch.device(device or "cuda")
        self.P, self.side = P, side
        self.H, self.W = (int(v) for v in A.input_dims)
        self.mode = mode
        self.guard = guard
        self.sigma = max(config.sigma, SIGMA_FLOOR_8BIT) / 255.0
        self.op = DeviceOperator(A)
        self.l2sq = None
        if lam is None:
            self.lam, self.l2sq = self.op.lambda_param(self.sigma)
        else:
            self.lam = float(lam)
        self.betas = beta_schedule(self.sigma, self.lam, config.beta_multipliers)
        self.plan = DevicePlan(model, tree, self.betas, with_tc=(mode == "tensor"))
        # per-plan kernel choices (bitwise-equivalent variants; fepll_plan_set_option)
        self.options = dict(options or {})
        for k, v in self.options.items():
            self.plan.set_option(k, v)
        self._agg_variant = self.plan.get_option("aggregate_variant")
        # a model with a positive score weight has no pre-scaled tcgen05 images:
        # its tree walk runs on the exact FP64 scorer (the same labels)
        self._select_mode = self.MODES[mode] if (mode == "exact" or self.plan.has_tc) else 0
        dev = self.device
        # sampling plans: generated on the device (csrc/grid.cu), bitwise the
        # reference's numpy Philox draws (patches.py:102-132)
        self._grids = [self._grid(t) for t in range(config.iterations)]
        self.anchors = [g[0] for g in self._grids]
        n = int(self.anchors[0].shape[0])
        self.n = n
        # per-pixel cover lists of each plan (shared by the whole batch)
        # (batches share them; a row strip or a large single image reuses them
        # across restores of the same plan — the gather over them is ~2x the
        # speed of the candidate search; small single images search directly)
        # Cover-list entries pack (patch << 8 | offset) in 31 bits: planes of
        # 2^23 or more patches (8192^2 at spacing 2, 3000^2 at spacing 1)
        # gather by candidate search instead, which has no such limit.
        n_loc_rows = (self.strip.a_hi - self.strip.a_lo + 1) if self.strip is not None else \
            self._grids[0][1]
        self._use_cover = ((self.batch > 1 or self.strip is not None
                            or self.H * self.W >= (4 << 20))
                           and n_loc_rows * self._grids[0][2] < (1 << 23))
        self._covers = [self._cover(t) if self._use_cover else self._cover_rows()
                        for t in range(config.iterations)]
        self.plan.reserve(n * self.batch)
        B, H, W = self.batch, self.H, self.W
        f64 = torch.float64
        self.z32_pitch = ((P + 31) // 32) * 32
        # FP64 patch rows (kernel (a) output) feed the DMMA Wiener kernel —
        # unless it reads the image windows itself (P = 64): allocated on
        # first need (_z64)
        self.Z64 = None
        # FP32 patch rows (kernel (a) output) feed the tensor-core scorer
        self.Z32 = (torch.empty((B * n, self.z32_pitch), dtype=torch.float32, device=dev)
                    if mode == "tensor" or precision == "fp32-state" else None)
        # Wiener output rows (est + dc), zhat_rows per image (the ABI allows a
        # padded pitch; a padded one measured no different, so dense)
        self.zhat_rows = n
        self._agg_dc = None  # traces: dc added by the gather (the Wiener kernel writes bare estimates)
        self.Zhat = torch.empty((B * self.zhat_rows, P), device=dev,
                                dtype=torch.float32 if precision == "fp32-state" else f64)
        self.dc = torch.empty(B * n, dtype=f64, device=dev)
        self.sq = torch.empty(B * n, dtype=f64, device=dev)
        self.labels = torch.empty(B * n, dtype=torch.int32, device=dev)
        self.leaf_counts = torch.zeros((config.iterations, len(model.components)), dtype=torch.int64,
                                       device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.rescored = torch.zeros((config.iterations, 64), dtype=torch.int32, device=dev)
        self._ts = None        # torch stream of the current run (event marks)
        self._tg_graph = None  # timed CUDA graph of restore() (capture_timed)
        self.use_graph = True  # restore() replays a captured graph when the plan is cached
        self._wcost = None     # per-component Wiener cost (counters)
        self.x = torch.empty((B, H, W), dtype=f64, device=dev)
        self._y_in = None  # identity restores: the observation, read in place
        self._force_z64 = False
        self._want_xt = False
        self.graph = None
        self.xt = torch.empty((B, H, W), dtype=f64, device=dev)
        kind = A.kind
        self.diag = None
        if kind in ("mask", "gain"):
            pm = np.asarray(A.pixel_map, dtype=np.float64)
            d = (pm != 0).astype(np.float64) if kind == "mask" else pm * pm
            self.diag = torch.from_numpy(d).to(dev).expand(B, H, W).contiguous()
        # batches with aggregate_variant 2: the cover lists re-addressed into
        # per-tile shared-memory stages (csrc/aggregate_tiles.cu)
        self._tiles = [self._tile_tables(t) for t in range(config.iterations)]
        self.aty = torch.empty((B, H, W), dtype=f64, device=dev)
        self.pixel_kind = A.solve_strategy == "pixel_diagonal"
        # rhs of the FFT / CG image update and the solver infos
        self.rhs = None if self.pixel_kind else torch.empty((B, H, W), dtype=f64, device=dev)
        self.solve_info = torch.zeros((config.iterations, B, 4), dtype=f64, device=dev)
        self.init_info = torch.zeros((B, 4), dtype=f64, device=dev)

    # ---------------------------------------------------------------- setup
    def _grid(self, t: int):
        """(device anchors [n][2] int32, n_rows, n_cols, half) of iteration t."""
        torch = self.torch
        c = self.config
        H, W, s, side = self.H, self.W, c.spacing, self.side
        jit = c.sampling == "jittered"
        half = (side - s) // 2 if jit else 0
        nr = axis_anchors(H, side, s).size
        nc = axis_anchors(W, side, s).size
        sp = self.strip
        if sp is not None:  # the global grid; this strip keeps nominal rows a_lo..a_hi
            H = sp.H
            nr = axis_anchors(H, side, s).size
        anchors = torch.empty((nr * nc, 2), dtype=torch.int32, device=self.device)
        scratch = torch.empty(N.lib().fepll_grid_scratch_ints(), dtype=torch.int32, device=self.device)
        status = torch.zeros(1, dtype=torch.int32, device=self.device)
        st = torch.cuda.current_stream(self.device).cuda_stream
        k0, k1 = philox_key(c.seed, t)
        N.call("fepll_sample_grid", k0, k1, H, W, side, s, int(jit), 0,
               N.ptr(anchors), N.ptr(scratch), N.ptr(status), st)
        if int(status.item()) & 4:
            raise NumericalError("sampling plan: more rejected Philox draws than the fix-up list holds")
        if sp is not None:
            anchors = anchors[sp.a_lo * nc:(sp.a_hi + 1) * nc].clone()
            anchors[:, 0] -= sp.slab_lo
        return anchors, nr, nc, half

    def _cover_rows(self):
        """(None, None, r0, r1): the produced rows, for the single-image path."""
        sp = self.strip
        if sp is None:
            return None, None, 0, self.H
        return None, None, sp.r0 - sp.slab_lo, sp.r1 - sp.slab_lo

    def _cover(self, t: int):
        """CSR cover lists (ptr, entries) of iteration t's plan for the rows
        this restorer produces (csrc/aggregate.cu fepll_cover_build)."""
        torch = self.torch
        anchors, nr, nc, half = self._grids[t]
        sp = self.strip
        if sp is None:
            row0, H_glob, a_first, n_loc_rows, r0, r1 = 0, self.H, 0, nr, 0, self.H
        else:
            row0, H_glob, a_first = sp.slab_lo, sp.H, sp.a_lo
            n_loc_rows, r0, r1 = sp.a_hi - sp.a_lo + 1, sp.r0 - sp.slab_lo, sp.r1 - sp.slab_lo
        npx = (r1 - r0) * self.W
        cap = n_loc_rows * nc * self.P
        dev = self.device
        ptr = torch.empty(npx + 1, dtype=torch.int32, device=dev)
        entries = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        scratch = torch.empty(int(N.lib().fepll_cover_scratch_ints(npx)), dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        N.call("fepll_cover_build", N.ptr(anchors), nr, nc, self.config.spacing, half, self.side,
               self.W, row0, H_glob, a_first, n_loc_rows, r0, r1, N.ptr(ptr), N.ptr(entries), cap,
               N.ptr(scratch), st)
        return ptr, entries, r0, r1

    def _tile_tables(self, t: int):
        """(seg_off, seg_cnt, cover16, seg_cap, max_seg) of iteration t's
        cover lists for fepll_aggregate_tiles (batches: several images in
        flight per CTA), or None (single images — one tile per CTA measured
        1.8x slower than the per-pixel gather at 8192^2, its copies not
        pipelined — the candidate-search path, other variants, or a plan
        whose tiles do not fit the tables: those keep the cover-list
        gather)."""
        if not (self._use_cover and self.batch > 1 and self._agg_variant == 2):
            return None
        torch = self.torch
        ptr, entries, r0, r1 = self._covers[t]
        _, _, _, half = self._grids[t]
        rows = r1 - r0
        tw = int(N.lib().fepll_tiles_width())
        n_tiles = rows * ((self.W + tw - 1) // tw)
        cap = int(N.lib().fepll_tiles_seg_cap(self.side, self.config.spacing, half))
        if cap * self.side > 65536 or n_tiles == 0:
            return None
        dev = self.device
        seg_off = torch.empty(n_tiles * cap, dtype=torch.int32, device=dev)
        seg_cnt = torch.empty(n_tiles, dtype=torch.int32, device=dev)
        cover16 = torch.empty(max(int(entries.numel()), 1), dtype=torch.int16, device=dev)
        max_cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        N.call("fepll_tiles_build", N.ptr(ptr), N.ptr(entries), self.P, self.side, self.W, rows, cap,
               N.ptr(seg_off), N.ptr(seg_cnt), N.ptr(cover16), N.ptr(max_cnt), N.ptr(status), st)
        if int(status.item()) != 0:
            return None
        max_seg = int(max_cnt.item())
        # the trace form stages dc too (the largest need), mask/gain a diagonal
        need = int(N.lib().fepll_tiles_smem_bytes(max_seg, self.side, 4 if self.precision == "fp32-state" else 8,
                                                  1, int(self.diag is not None)))
        if need > 200 * 1024:
            return None
        return seg_off, seg_cnt, cover16, cap, max_seg

    # ---------------------------------------------------------------- loop
    def run(self, y_dev, trace: bool = False, timer: dict | None = None, exchange=None):
        """y_dev: (B, Ho, Wo) float64 device tensor.  Returns x (B, H, W) on
        the device and the per-iteration records.  ``timer`` (optional dict)
        collects CUDA-event pairs per phase for profiling; ``exchange(t)``
        (strip mode) refreshes the halo rows after iteration t."""
        self.start(y_dev, timer)
        records = []
        for t in range(len(self.betas)):
            records.extend(self.iterate(t, trace, timer))
            if exchange is not None and t + 1 < len(self.betas):
                exchange(t)
        return self.x, records

    def start(self, y_dev, timer: dict | None = None) -> None:
        """x0 (solver.py:195-198) for a device-resident observation batch."""
        torch = self.torch
        self._ts = torch.cuda.current_stream(self.device)
        st = self._ts.cuda_stream
        A = self.A
        self.status.zero_()
        self._mark(timer, "start")
        self._y_in = None
        if A.kind == "identity":
            # solver.py:195-196: x0 = y; A^T y = y.  The observation buffer
            # itself serves as A^T y and as iteration 0's image (no copies);
            # strips keep copies (their halo rows are refreshed in place)
            if (self.strip is None and y_dev.dtype == torch.float64 and y_dev.is_contiguous()
                    and tuple(y_dev.shape) == tuple(self.x.shape) and y_dev.device == self.x.device):
                self._y_in = y_dev
            else:
                self.aty.copy_(y_dev)
                self.x.copy_(y_dev)
        else:
            cg = self.config.cg
            for b in range(self.batch):
                self.op.adjoint(y_dev[b], self.aty[b], st)
                # solver.py:198 -> operators.py:374-394
                self.op.init(y_dev[b], self.aty[b], self.sigma, self.lam, cg.tolerance,
                             cg.max_iterations, self.x[b], self.init_info[b], st)
        self._mark(timer, "init")

    def iterate(self, t: int, trace: bool = False, timer: dict | None = None) -> list:
        """One HQS iteration (solver.py:200-262); returns its trace record
        (empty unless ``trace``) with the reference's keys
        (`pkg/src/fepll/solver.py:258-266`): beta, grid (a SampleGrid),
        patches, dc, selected, estimates (the bare Wiener estimates, without
        dc), x_tilde — each with a leading batch axis — plus x."""
        ts = self.torch.cuda.current_stream(self.device) if timer is None or self._ts is None else self._ts
        self._ts = ts
        st = ts.cuda_stream
        self._want_xt = trace
        if not trace:
            self._iteration(t, st, timer)
            return []
        # trace: the Wiener kernel writes the bare estimates and the gather
        # adds dc (the same single FP64 rounding of patches.py:209, so x is
        # bitwise the untraced result); the FP64 patch rows are kept
        fp32 = self.precision == "fp32-state"
        if not fp32:
            self.plan.set_option("wiener_add_dc", 0)
            self._agg_dc = self.dc
        self._force_z64 = True
        try:
            self._iteration(t, st, timer)
        finally:
            if not fp32:
                self.plan.set_option("wiener_add_dc", self.options.get("wiener_add_dc", 1))
            self._agg_dc = None
            self._force_z64 = False
        B, n, P = self.batch, self.n, self.P
        est = self.Zhat.view(B, self.zhat_rows, P)[:, :n].double()
        if fp32:  # FP32 est + dc: the estimates up to that rounding
            est = est - self.dc.view(B, n, 1)
        return [{"beta": float(self.betas[t]),
                 "grid": self.sample_grid(t),
                 "patches": self.Z64.view(B, n, P).cpu().numpy().copy(),
                 "dc": self.dc.view(B, n).cpu().numpy().copy(),
                 "selected": self.labels.view(B, n).cpu().numpy().astype(np.int64),
                 "estimates": est.cpu().numpy().copy(),
                 "x_tilde": self.xt.cpu().numpy().copy(),
                 "x": self.x.cpu().numpy().copy()}]

    def sample_grid(self, t: int) -> SampleGrid:
        """Iteration t's sampling plan as the reference's SampleGrid
        (`pkg/src/fepll/patches.py:40-69`): positions from the device
        generator; the host generator supplies offsets and global_shift."""
        c = self.config
        H, W = self.H, self.W
        if self.strip is not None:
            H = self.strip.H
        if c.sampling == "jittered":
            g = jittered_grid(H, W, self.P, c.spacing, jitter_rng(c.seed, t))
        else:
            g = regular_grid(H, W, self.P, c.spacing)
        pos = self.anchors[t].cpu().numpy().astype(np.int64)
        if self.strip is None and not np.array_equal(pos, g.positions):
            raise N.DeviceError("device sampling plan differs from the reference generator")
        return SampleGrid(pos, (self.H, self.W), g.patch_side, g.spacing, g.mode,
                          offsets=g.offsets, global_shift=g.global_shift)

    def _mark(self, timer, name):
        if timer is None:
            return
        stamps = timer.get("_stamps")
        if stamps is not None:
            # graph capture (capture_timed): a device timestamp kernel per mark
            names = timer.setdefault("_names", [])
            if len(names) >= stamps.numel():
                raise DeviceError("timestamp buffer too small for this restore")
            N.call("fepll_stamp", stamps.data_ptr() + 8 * len(names), self._ts.cuda_stream)
            names.append(name)
            return
        ev = self.torch.cuda.Event(enable_timing=True)
        # the stream object is looked up once per run (start()): torch's
        # current_stream() costs ~15 us a call, 27 marks per restore
        ts = self._ts
        if ts is None:
            ev.record()
        else:
            ev.record(ts)
        timer.setdefault("_marks", []).append((name, ev))

    def _iteration(self, t: int, st, timer=None) -> None:
        B, H, W, P, side = self.batch, self.H, self.W, self.P, self.side
        anchors, nr, nc, half = self._grids[t]
        n = self.n
        nt = B * n
        mode = self._select_mode
        self._mark(timer, "start")
        # iteration 0 of an identity restore reads the observation in place
        xin = self._y_in if (t == 0 and self._y_in is not None) else self.x
        aty = self._y_in if self._y_in is not None else self.aty
        z64 = self._z64()
        N.call("fepll_extract", N.ptr(xin), B, H, W, side, N.ptr(anchors), n, nc,
               N.ptr(z64), N.ptr(self.Z32), self.z32_pitch, N.ptr(self.dc), N.ptr(self.sq), st)
        self._mark(timer, "extract")
        N.call("fepll_select", self.plan.handle, t, N.ptr(xin), H, W, N.ptr(anchors), n,
               N.ptr(self.dc), N.ptr(self.sq), N.ptr(self.Z32), N.ptr(z64), nt, mode,
               float(self.guard),
               N.ptr(self.labels), N.ptr(self.leaf_counts[t]), st)
        N.call("fepll_select_rescored", self.plan.handle, N.ptr(self.rescored[t]), st)
        self._mark(timer, "select")
        if self.precision == "fp32-state":
            N.call("fepll_wiener_f32", self.plan.handle, t, N.ptr(xin), H, W, N.ptr(anchors), n,
                   N.ptr(self.dc), N.ptr(self.Z32), self.z32_pitch, nt, N.ptr(self.Zhat), self.zhat_rows, st)
        else:
            N.call("fepll_wiener", self.plan.handle, t, N.ptr(xin), H, W, N.ptr(anchors), n,
                   N.ptr(self.dc), N.ptr(z64), nt, N.ptr(self.Zhat), self.zhat_rows, st)
        self._mark(timer, "wiener")
        bs2 = float(self.betas[t]) * self.sigma * self.sigma
        # reproject (patches.py:198-222; Zhat already holds est + dc, so the
        # gathers get no dc); pixel-diagonal kinds fuse the image
        # update (operators.py:281-287), the others get rhs = A^T y + bs2 x~ for
        # the FFT / CG solve.  Batches, strips and large images gather over
        # the plan's cover lists; small single images search their candidates
        # directly.
        ptr, entries, r0, r1 = self._covers[t]
        sfx = "_f32" if self.precision == "fp32-state" else ""
        kind = 0 if self.pixel_kind else 1
        out = self.x if self.pixel_kind else self.rhs
        diag = self.diag if self.pixel_kind else None
        xt = self.xt if (self._want_xt or not self.pixel_kind) else None
        if not self._use_cover:
            sp = self.strip
            row0, H_glob, a_first, n_loc = ((sp.slab_lo, sp.H, sp.a_lo, sp.a_hi - sp.a_lo + 1)
                                            if sp is not None else (0, H, 0, nr))
            N.call("fepll_aggregate_strip" + sfx, N.ptr(self.Zhat), N.ptr(self._agg_dc), N.ptr(anchors), nr, nc,
                   self.config.spacing, half, side, B, H, W, row0, H_glob, a_first, n_loc, r0, r1,
                   N.ptr(aty), N.ptr(diag), bs2, kind, N.ptr(out), N.ptr(xt), N.ptr(self.status), st)
        elif self._tiles[t] is not None:
            z64, z32 = (None, self.Zhat) if sfx else (self.Zhat, None)
            seg_off, seg_cnt, cover16, cap, max_seg = self._tiles[t]
            N.call("fepll_aggregate_tiles", N.ptr(z64), N.ptr(z32), N.ptr(self._agg_dc), n, N.ptr(ptr),
                   N.ptr(cover16),
                   N.ptr(seg_off), N.ptr(seg_cnt), cap, max_seg, P, self.zhat_rows, B, H, W, r0, r1,
                   N.ptr(aty), N.ptr(diag), bs2, kind, N.ptr(out), N.ptr(xt), N.ptr(self.status), st)
        else:
            z64, z32 = (None, self.Zhat) if sfx else (self.Zhat, None)
            N.call("fepll_aggregate_cover_ex", N.ptr(z64), N.ptr(z32), N.ptr(self._agg_dc), N.ptr(ptr),
                   N.ptr(entries), P, n, self.zhat_rows, B, H, W, r0, r1, N.ptr(aty), N.ptr(diag), bs2, kind,
                   N.ptr(out), N.ptr(xt), N.ptr(self.status), self._agg_variant % 2, st)
        self._mark(timer, "aggregate")
        if not self.pixel_kind:
            cg = self.config.cg
            for b in range(B):
                self.op.solve(self.rhs[b], self.xt[b], bs2, cg.tolerance, cg.max_iterations,
                              self.x[b], self.solve_info[t, b], self.status, st)
            self._mark(timer, "image_solve")

    def _z64(self):
        """The FP64 patch rows, or None when nothing needs them: the Wiener
        kernel reads the image windows (plan option wiener_xw) or the FP32
        rows (fp32-state), and no trace wants them (the re-scoring then
        re-extracts the FP64 patches from the image)."""
        if ((self.precision == "fp32-state" or N.lib().fepll_wiener_reads_image(self.plan.handle))
                and not self._force_z64):
            return None
        if self.Z64 is None:
            self.Z64 = self.torch.empty((self.batch * self.n, self.P), dtype=self.torch.float64,
                                        device=self.device)
        return self.Z64

    # reference names of the phases (pkg/src/fepll/solver.py:206-254)
    PHASE_NAMES = {"extract": "extract", "select": "select", "wiener": "estimate",
                   "aggregate": "reproject", "image_solve": "image_solve"}

    @staticmethod
    def phase_times(timer: dict) -> dict:
        """Milliseconds per phase from the marks recorded by run().  Every
        interval between consecutive marks is attributed: the stretch before
        an iteration's first mark (host launch gaps between iterations)
        counts as "gap", so the phases add up to the run's span."""
        out: dict = {}
        marks = timer.get("_marks", [])
        for ((n0, e0), (n1, e1)), ms in zip(zip(marks, marks[1:]), Restorer._mark_ms(timer)):
            key = "gap" if n1 == "start" else n1
            out[key] = out.get(key, 0.0) + ms
        return out

    @staticmethod
    def _mark_ms(timer: dict) -> list:
        """Milliseconds between consecutive marks (read once per timer)."""
        marks = timer.get("_marks", [])
        ms = timer.get("_ms")
        if ms is None or len(ms) != max(0, len(marks) - 1):
            ms = [e0.elapsed_time(e1) for (_, e0), (_, e1) in zip(marks, marks[1:])]
            timer["_ms"] = ms
        return ms

    @classmethod
    def iteration_times(cls, timer: dict) -> list:
        """Seconds per phase of each HQS iteration, under the reference's
        ``IterationStats.times`` keys (grid, extract, select, estimate,
        reproject, image_solve).  The sampling plans are part of the cached
        device plan (generated once, csrc/grid.cu), so "grid" is 0.  For the
        pixel-diagonal kinds the image update is fused into the gather and
        its time is inside "reproject"."""
        out = []
        marks = timer.get("_marks", [])
        cur = None
        for ((n0, e0), (n1, e1)), ms in zip(zip(marks, marks[1:]), cls._mark_ms(timer)):
            if n1 == "start":
                continue
            if n1 == "extract":
                cur = {"grid": 0.0}
                out.append(cur)
            if cur is None or n1 not in cls.PHASE_NAMES:
                continue
            cur[cls.PHASE_NAMES[n1]] = ms / 1e3
        return out

    # ---------------------------------------------------------------- graphs
    def capture(self, y_dev):
        """Record one whole restore (x0 + every iteration) of the device
        observation buffer ``y_dev`` as a CUDA graph; :meth:`replay` re-runs
        it (refill ``y_dev`` in place between replays).  The C ABI is
        stream-ordered with no host synchronisation, so the captured launch
        sequence is exactly :meth:`run`'s.  Returns the output tensor."""
        torch = self.torch
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):  # warm-up off the capture (lazy allocations)
            self.run(y_dev)
        torch.cuda.current_stream(self.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            x, _ = self.run(y_dev)
        self._graph_y = y_dev
        return x

    def replay(self):
        self.graph.replay()
        return self.x

    def capture_timed(self):
        """As :meth:`capture` on an observation buffer owned by the restorer,
        with a device timestamp (``fepll_stamp``) at every phase mark, so a
        replay still yields the per-phase times of that call."""
        torch = self.torch
        self._tg_y = torch.zeros((self.batch,) + tuple(self.A.output_dims), dtype=torch.float64,
                                 device=self.device)
        self._tg_stamps = torch.zeros(16 + 8 * len(self.betas), dtype=torch.int64, device=self.device)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):  # warm-up off the capture (lazy allocations)
            self.run(self._tg_y)
        torch.cuda.current_stream(self.device).wait_stream(side)
        timer = {"_stamps": self._tg_stamps}
        self._tg_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._tg_graph):
            self.run(self._tg_y, timer=timer)
        self._tg_names = list(timer["_names"])

    def run_timed_graph(self, ys_host):
        """Upload ``ys_host`` (B, Ho, Wo float64 numpy), replay the timed
        graph and return (x on the device, timer) — the timer carries the
        phase names and the milliseconds between consecutive marks, the form
        :meth:`phase_times` / :meth:`iteration_times` read."""
        torch = self.torch
        if getattr(self, "_tg_graph", None) is None:
            self.capture_timed()
        self._tg_y.copy_(torch.from_numpy(ys_host))
        self._tg_graph.replay()
        st = self._tg_stamps[:len(self._tg_names)].cpu().numpy()
        ms = [float(b - a) / 1e6 for a, b in zip(st[:-1], st[1:])]
        return self.x, {"_marks": [(n, None) for n in self._tg_names], "_ms": ms}

    def counters(self):
        """(patches, evals, selection mults, estimation mults) per iteration
        from the label histograms (every leaf has one root path)."""
        hist = self.leaf_counts.cpu().numpy()
        P = self.P
        if self._wcost is None:
            self._wcost = np.array([wiener_flat_cost(c.kept_basis.shape[1], P) for c in self.model.components])
        wcost = self._wcost
        out = []
        for t in range(hist.shape[0]):
            h = hist[t]
            out.append((int(h.sum()), int(h @ self.plan.path_evals), int(h @ self.plan.path_mults),
                        int(h @ wcost)))
        return out

    def check_status(self, t_last: int | None = None, rescored_host=None):
        s = int(self.status.item())
        if s & 1:
            raise DataError("reprojection target has uncovered pixels")
        if s & 2:
            raise NumericalError("non-finite image estimate")
        rs = self.rescored.cpu().numpy() if rescored_host is None else rescored_host
        if int(rs[:, 63].max()) != 0:  # csrc/select.cu deferred verification
            raise DeviceError("deferred verification ran out of log or leaf-bucket slots")
        if not self.pixel_kind and self.A.kind == "decimate":
            finite = self.solve_info[:, :, 3].cpu().numpy()
            if np.any(finite == 0):
                raise NumericalError("non-finite image estimate")

    def solve_infos(self):
        """(converged, residual) per iteration (first image), the
        `SolveInfo` fields the reference records (solver.py:252-253)."""
        if self.pixel_kind or self.A.kind == "convolution":
            return [(True, 0.0)] * len(self.betas)
        si = self.solve_info.cpu().numpy()
        return [(bool(si[t, 0, 2] > 0), float(si[t, 0, 1])) for t in range(si.shape[0])]


class HostPipeline:
    """Batch restoration from and to pinned host buffers with the copies
    overlapped: the batch is cut into ``chunks`` equal parts that rotate over
    ``streams`` restorers, one CUDA stream each, so the upload of chunk c+1
    and the download of chunk c-1 run on the copy engines while chunk c
    computes — across consecutive :meth:`submit` calls too (a stream of
    batches; with chunks=1 every batch keeps the full-batch kernel
    efficiency and its copies hide behind its neighbours' compute).
    Results are identical to :class:`Restorer` on the whole batch (every
    image is restored independently)."""

    def __init__(self, A, model, tree, config, batch: int, chunks: int = 1, lam: float | None = None,
                 mode: str = "tensor", device=None, streams: int = 2, graphs: bool = False,
                 precision: str = "fp64", options: dict | None = None):
        torch = _torch()
        if batch % chunks:
            raise DataError(f"batch {batch} does not split into {chunks} chunks")
        self.torch = torch
        self.batch, self.chunks = int(batch), int(chunks)
        self.per = self.batch // self.chunks
        k = max(1, int(streams))  # restorers / streams the chunks rotate over
        self.restorers = [Restorer(A, model, tree, config, batch=self.per, lam=lam, mode=mode,
                                   device=device, precision=precision, options=options)
                          for _ in range(k)]
        dev = self.restorers[0].device
        self.device = dev
        self.streams = [torch.cuda.Stream(dev) for _ in range(k)]
        Ho, Wo = (int(v) for v in A.output_dims)
        H, W = (int(v) for v in A.input_dims)
        self.y32 = [torch.empty((self.per, Ho, Wo), dtype=torch.float32, device=dev) for _ in range(k)]
        self.y64 = [torch.empty((self.per, Ho, Wo), dtype=torch.float64, device=dev) for _ in range(k)]
        self.x32 = [torch.empty((self.per, H, W), dtype=torch.float32, device=dev) for _ in range(k)]
        self.status = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(k)]
        # graphs: each restorer's whole restore of its y64 buffer is captured
        # once and replayed per chunk (one launch instead of ~100)
        self.graphs = bool(graphs)
        if self.graphs:
            for yb, r in zip(self.y64, self.restorers):
                yb.zero_()
                r.capture(yb)
            torch.cuda.synchronize(dev)
        self._next = 0  # chunk counter: chunk j runs on restorer / stream j % k
        self._computed = None  # event: the last queued chunk's compute is done

    def submit(self, y_host, x_host) -> None:
        """Queue one batch without waiting: y_host pinned (batch, Ho, Wo)
        float32 observations, x_host pinned (batch, H, W) float32 output.
        Chunks keep rotating over the streams across calls, so the copies of
        one batch overlap the compute of its neighbours (with chunks=1, batch
        s+1 uploads while batch s computes); neither buffer may be touched
        until :meth:`wait` returns."""
        torch = self.torch
        main = torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(main)
        for c in range(self.chunks):
            k = self._next % len(self.restorers)
            self._next += 1
            r, s = self.restorers[k], self.streams[k]
            lo, hi = c * self.per, (c + 1) * self.per
            with torch.cuda.stream(s):
                self.y32[k].copy_(y_host[lo:hi], non_blocking=True)
                self.y64[k].copy_(self.y32[k])
                # computes run one after another (two restorations sharing
                # the SMs measured slower than back to back); only the copies
                # overlap them
                if self._computed is not None:
                    s.wait_event(self._computed)
                x = r.replay() if self.graphs else r.run(self.y64[k])[0]
                self._computed = torch.cuda.Event()
                self._computed.record(s)
                self.x32[k].copy_(x)
                x_host[lo:hi].copy_(self.x32[k], non_blocking=True)
                self.status[k].bitwise_or_(r.status)  # run() clears it per chunk

    def join(self) -> None:
        """Make the current stream wait for every queued batch (no host sync)."""
        main = self.torch.cuda.current_stream(self.device)
        for s in self.streams:
            main.wait_stream(s)

    def wait(self) -> None:
        """Block until every queued batch is in its host buffer; raise on a
        numerical / coverage error of any of them."""
        self.join()
        self.torch.cuda.current_stream(self.device).synchronize()
        for r, st in zip(self.restorers, self.status):
            r.status.copy_(st)
            st.zero_()
            r.check_status()

    def run(self, y_host, x_host) -> None:
        """submit() + wait(): returns after the batch is restored into x_host."""
        self.submit(y_host, x_host)
        self.wait()


# ------------------------------------------------------------------ plan cache
_CACHE_SIZE = 4
_restorer_cache: "OrderedDict[tuple, tuple]" = None  # key -> (Restorer, pinned key objects)


def _array_digest(a) -> str:
    if a is None:
        return ""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha1(a.tobytes()).hexdigest() + str(a.shape)


def _plan_key(A, model, tree, config, batch, lam, mode, options, precision="fp64"):
    """Cache key of a Restorer: model and tree by identity (immutable and
    shareable; the cache pins them so an id is never
    reused while cached), the operator by value (kind, dims, factor, kernel
    and pixel-map bytes), every config field that shapes the plan."""
    cg = config.cg
    op = (A.kind, tuple(A.input_dims), tuple(A.output_dims), getattr(A, "factor", None),
          _array_digest(getattr(A, "kernel", None)), _array_digest(getattr(A, "pixel_map", None)))
    cfg = (float(config.sigma), int(config.iterations), tuple(float(v) for v in config.beta_multipliers),
           int(config.spacing), config.sampling, bool(config.use_tree), bool(config.use_flat_tail),
           int(config.seed), float(cg.tolerance), int(cg.max_iterations))
    return (id(model), id(tree), op, cfg, int(batch), None if lam is None else float(lam), mode,
            tuple(sorted((options or {}).items())), precision)


def cached_restorer(A, model, tree, config, batch: int = 1, lam=None, mode: str = "tensor",
                    options: dict | None = None, precision: str = "fp64") -> "Restorer":
    """The Restorer for these arguments, built once and reused by later
    :func:`restore` / :func:`restore_batch` calls (plan packing, lambda,
    sampling plans, cover lists and scratch are the per-call setup the
    reference redoes every call).  Least-recently-used, 4 entries."""
    global _restorer_cache
    if _restorer_cache is None:
        _restorer_cache = OrderedDict()
    key = _plan_key(A, model, tree, config, batch, lam, mode, options, precision)
    hit = _restorer_cache.get(key)
    if hit is not None:
        _restorer_cache.move_to_end(key)
        return hit[0]
    r = Restorer(A, model, tree, config, batch=batch, lam=lam, mode=mode, options=options,
                 precision=precision)
    _restorer_cache[key] = (r, (model, tree))
    while len(_restorer_cache) > _CACHE_SIZE:
        _restorer_cache.popitem(last=False)
    return r


def clear_plan_cache() -> None:
    global _restorer_cache
    _restorer_cache = None


def restore(y, A, model, tree=None, config=None, *, mode: str = "tensor", lam=None,
            options: dict | None = None, precision: str = "fp64"):
    """GPU drop-in for `pkg/src/fepll/solver.py:161-274`: same signature,
    validations, errors, counters, ``IterationStats.times`` and trace
    records (one image, no batch axis)."""
    if config is None:
        config = RestorationConfig(sigma=20.0)
    _validate_config(config)
    y = np.asarray(y, dtype=np.float64)
    if tuple(y.shape) != tuple(A.output_dims):
        raise DataError(f"observation shape {y.shape} != operator output {tuple(A.output_dims)}")
    x, stats = restore_batch(y[None], A, model, tree, config, mode=mode, lam=lam, options=options,
                             precision=precision)
    if config.trace:
        for rec in stats.trace:
            for k in ("patches", "dc", "selected", "estimates", "x_tilde", "x"):
                rec[k] = rec[k][0]
    return x[0], stats


def restore_batch(ys, A, model, tree=None, config=None, *, mode: str = "tensor", lam=None,
                  restorer: Restorer | None = None, options: dict | None = None,
                  precision: str = "fp64"):
    """Restore a (B, H, W) stack sharing operator, sigma and seed.  The
    device plan comes from the plan cache unless ``restorer`` is given."""
    if config is None:
        config = RestorationConfig(sigma=20.0)
    t0 = time.perf_counter()
    ys = np.asarray(ys, dtype=np.float64)
    if ys.ndim != 3:
        raise DataError("restore_batch expects a (B, H, W) stack")
    if tuple(ys.shape[1:]) != tuple(A.output_dims):
        raise DataError(f"observation shape {ys.shape[1:]} != operator output {tuple(A.output_dims)}")
    r = restorer or cached_restorer(A, model, tree, config, batch=ys.shape[0], lam=lam, mode=mode,
                                    options=options, precision=precision)
    if r.batch != ys.shape[0]:
        raise DataError(f"restorer batch {r.batch} != {ys.shape[0]} observations")
    torch = r.torch
    if restorer is None and not config.trace and r.strip is None and r.use_graph:
        # cached plan, no trace: one CUDA-graph replay of the whole restore
        # (device timestamps keep IterationStats.times per call)
        t1 = time.perf_counter()
        x_dev, timer = r.run_timed_graph(np.ascontiguousarray(ys))
        recs = []
    else:
        y_dev = torch.from_numpy(np.ascontiguousarray(ys)).to(r.device)
        t1 = time.perf_counter()
        timer = {}
        x_dev, recs = r.run(y_dev, trace=config.trace, timer=timer)
    x = x_dev.cpu().numpy()
    rescored = r.rescored.cpu().numpy()
    r.check_status(rescored_host=rescored)
    stats = SolverStats(lam=r.lam)
    phases = Restorer.phase_times(timer)
    stats.init_seconds = (t1 - t0) + phases.get("init", 0.0) / 1e3
    infos = r.solve_infos()
    times = Restorer.iteration_times(timer)
    for t, (npatch, ev, sm, em) in enumerate(r.counters()):
        it = IterationStats(beta=float(r.betas[t]), patches=npatch // max(r.batch, 1),
                            image_solve_converged=infos[t][0], image_solve_residual=infos[t][1],
                            score_evaluations=ev, selection_multiplies=sm,
                            estimation_multiplies=em,
                            times=times[t] if t < len(times) else {})
        stats.iterations.append(it)
    stats.trace = recs
    stats.rescored = [int(v) for v in rescored[:, :62].sum(axis=1)]
    stats.repaired = [int(v) for v in rescored[:, 62]]
    stats.total_seconds = time.perf_counter() - t0
    return x, stats
