"""Strip mode: one large denoising image split by pixel rows across ranks.

SURVEY §8(e), cfg5 strip: rank g owns pixel rows [r0, r1).  It processes
every anchor of the global sampling plan whose nominal row can cover an owned
pixel (the candidate rows of the reprojection gather, patches.py:198-222), so
it holds a slab of the image — its owned rows plus halo rows above and below
(at most side - 1 + half each side).  Per HQS iteration:

* extraction / selection / Wiener run on the slab's anchors (every patch is
  computed exactly as in the unsplit run — per-patch arithmetic does not
  depend on which other patches share a launch);
* the reprojection gather and the pixel update (solver.py x-update for the
  identity operator) produce the owned rows only, visiting the same global
  candidates in the same order — owned pixels are bit-identical to the
  unsplit run;
* the halo rows of the next iteration's slab are refreshed from the ranks
  owning them (:func:`exchange_halos`: grouped point-to-point sends /
  receives — NCCL on GPUs, gloo in the CPU tests).

x0 = y (solver.py:195-196) needs no communication, and lambda / beta are
identical on every rank.  Deblur / SR (global FFT or CG solves) do not split
by rows: they run as replicas.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import DataError
from .patches import axis_anchors

__all__ = ["batch_shard", "StripSpec", "strip_rows", "strip_spec", "strip_specs", "halo_plan",
           "exchange_halos", "StripRestorer", "restore_strips_single_process"]


def batch_shard(n_images: int, world: int, rank: int) -> list:
    """cfg5 batch mode: images are independent, rank g
    restores a contiguous block of n/world of them — no data-path
    collective.  n_images must split evenly."""
    if world < 1 or not 0 <= rank < world:
        raise DataError("bad rank / world size")
    if n_images % world:
        raise DataError(f"{n_images} images do not split over {world} ranks")
    per = n_images // world
    return list(range(rank * per, (rank + 1) * per))


@dataclass(frozen=True)
class StripSpec:
    H: int              # global image rows
    W: int
    r0: int             # owned global pixel rows [r0, r1)
    r1: int
    slab_lo: int        # global rows held locally [slab_lo, slab_hi)
    slab_hi: int
    a_lo: int           # global nominal anchor rows processed, inclusive
    a_hi: int
    n_rows: int         # global nominal grid
    n_cols: int

    @property
    def slab_rows(self) -> int:
        return self.slab_hi - self.slab_lo


def strip_rows(H: int, world: int, rank: int) -> tuple:
    """Even split of the pixel rows."""
    if not 0 <= rank < world or world > H:
        raise DataError("bad strip rank / world size")
    return rank * H // world, (rank + 1) * H // world


def _ceil_div0(num: int, s: int) -> int:
    return 0 if num <= 0 else -(-num // s)


def strip_spec(H: int, W: int, patch_dim: int, spacing: int, half: int, r0: int, r1: int) -> StripSpec:
    """Anchor rows and slab of the strip owning pixel rows [r0, r1).  The
    candidate rows mirror the gather of csrc/aggregate.cu: nominal rows a with
    a*s in [r - side + 1 - half, r + half] (a <= n_rows - 2) plus the clamped
    last row when H - side <= r + half."""
    side = math.isqrt(patch_dim)
    if side * side != patch_dim:
        raise DataError(f"patch_dim {patch_dim} is not a perfect square")
    if not 0 <= r0 < r1 <= H:
        raise DataError("strip rows outside the image")
    n_rows = axis_anchors(H, side, spacing).size
    n_cols = axis_anchors(W, side, spacing).size
    last_r = H - side
    a_lo = min(_ceil_div0(r0 - side + 1 - half, spacing), n_rows - 1)
    a_hi = min(n_rows - 2, (r1 - 1 + half) // spacing)
    if last_r <= r1 - 1 + half:
        a_hi = n_rows - 1
    a_hi = max(a_hi, a_lo)

    def nominal(a):
        return last_r if a == n_rows - 1 else a * spacing

    slab_lo = max(0, nominal(a_lo) - half)
    slab_hi = min(H, nominal(a_hi) + half + side)
    if not (slab_lo <= r0 and r1 <= slab_hi):
        raise DataError("strip slab does not cover its owned rows")
    return StripSpec(H, W, r0, r1, slab_lo, slab_hi, a_lo, a_hi, n_rows, n_cols)


def strip_specs(H: int, W: int, patch_dim: int, spacing: int, half: int, world: int) -> list:
    return [strip_spec(H, W, patch_dim, spacing, half, *strip_rows(H, world, g)) for g in range(world)]


def halo_plan(specs: list, rank: int) -> list:
    """[(peer, send_rows, recv_rows)] in global rows, (lo, hi) or None:
    receive the slab rows the peer owns, send the owned rows in the peer's
    slab.  Peers in ascending rank order (the same order on every rank)."""
    me = specs[rank]
    out = []
    for q, sq in enumerate(specs):
        if q == rank:
            continue
        lo, hi = max(me.slab_lo, sq.r0), min(me.slab_hi, sq.r1)
        recv = (lo, hi) if lo < hi else None
        lo, hi = max(sq.slab_lo, me.r0), min(sq.slab_hi, me.r1)
        send = (lo, hi) if lo < hi else None
        if send or recv:
            out.append((q, send, recv))
    return out


def exchange_halos(x_slab, specs: list, rank: int, group=None) -> None:
    """Refresh the halo rows of this rank's slab ([slab_rows][W], contiguous
    device or host tensor) with one grouped batch of point-to-point sends and
    receives (torch.distributed: NCCL / gloo)."""
    import torch.distributed as dist

    me = specs[rank]
    ops = []
    for q, send, recv in halo_plan(specs, rank):
        if send:
            ops.append(dist.P2POp(dist.isend, x_slab[send[0] - me.slab_lo:send[1] - me.slab_lo], q, group))
        if recv:
            ops.append(dist.P2POp(dist.irecv, x_slab[recv[0] - me.slab_lo:recv[1] - me.slab_lo], q, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class StripRestorer:
    """The restoration loop of one strip (wraps :class:`solver.Restorer`)."""

    def __init__(self, H: int, W: int, model, tree, config, rank: int, world: int,
                 mode: str = "tensor", device=None, lam: float | None = None,
                 precision: str = "fp64", options: dict | None = None):
        from .operators import identity_operator
        from .solver import Restorer

        side = math.isqrt(int(model.patch_dim))
        half = (side - config.spacing) // 2 if config.sampling == "jittered" else 0
        self.specs = strip_specs(H, W, int(model.patch_dim), config.spacing, half, world)
        self.spec = self.specs[rank]
        self.rank, self.world = rank, world
        sp = self.spec
        if lam is None:
            # lambda of the whole image's operator (operators.py:342-355), so
            # every strip runs the unsplit beta schedule bit for bit
            from .device_ops import DeviceOperator
            from .solver import SIGMA_FLOOR_8BIT
            lam, _ = DeviceOperator(identity_operator((H, W))).lambda_param(
                max(config.sigma, SIGMA_FLOOR_8BIT) / 255.0)
        self.restorer = Restorer(identity_operator((sp.slab_rows, W)), model, tree, config, batch=1,
                                 lam=lam, mode=mode, device=device, strip=sp, precision=precision,
                                 options=options)

    def run(self, y_slab_dev, group=None, timer=None):
        """y_slab_dev: (1, slab_rows, W) device tensor of the observation's
        slab rows.  Returns the owned rows (r1 - r0, W) of x on the device."""
        r = self.restorer

        def exchange(t):
            exchange_halos(r.x[0], self.specs, self.rank, group)

        x, _ = r.run(y_slab_dev, timer=timer, exchange=exchange if self.world > 1 else None)
        sp = self.spec
        return x[0, sp.r0 - sp.slab_lo:sp.r1 - sp.slab_lo]


def restore_strips_single_process(y, model, tree, config, world: int, mode: str = "tensor"):
    """All strips of one image on one device, in lockstep, halos copied
    between the slabs directly — the host-side check that strip mode is
    bit-identical to the unsplit run (no rank waits on another)."""
    import torch

    y = np.asarray(y, dtype=np.float64)
    H, W = y.shape
    strips = [StripRestorer(H, W, model, tree, config, g, world, mode=mode) for g in range(world)]
    for s in strips:
        sp = s.spec
        s.restorer.start(torch.from_numpy(np.ascontiguousarray(y[None, sp.slab_lo:sp.slab_hi])).cuda())
    T = len(strips[0].restorer.betas)
    for t in range(T):
        for s in strips:
            s.restorer.iterate(t)
        if t + 1 < T:
            for g, s in enumerate(strips):
                me = s.spec
                for q, _, recv in halo_plan(s.specs, g):
                    if recv:
                        src = strips[q]
                        sq = src.spec
                        s.restorer.x[0, recv[0] - me.slab_lo:recv[1] - me.slab_lo].copy_(
                            src.restorer.x[0, recv[0] - sq.slab_lo:recv[1] - sq.slab_lo])
    out = np.empty((H, W))
    for s in strips:
        sp = s.spec
        s.restorer.check_status()
        out[sp.r0:sp.r1] = s.restorer.x[0, sp.r0 - sp.slab_lo:sp.r1 - sp.slab_lo].cpu().numpy()
    return out
