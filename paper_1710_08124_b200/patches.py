"""Sampling plans: regular and jittered anchor grids.

The anchor arithmetic restates `pkg/src/fepll/patches.py:79-132`:
anchors every ``spacing`` pixels with the last one clamped to ``extent-side``;
the jittered grid adds a global shift folded into the band
``[-half, half]`` (half = (side-spacing)//2), per-anchor jitter, clipping, and
pins the boundary anchors.  Draws come from
``Generator(Philox(key=[seed, t]))`` (`pkg/src/fepll/patches.py:102-104`).

Two producers exist for the jittered plan:

* :func:`jittered_grid` — host numpy (the same bit generator the reference
  uses); kept for plan inspection and the CPU tests;
* the device generator ``fepll_sample_grid`` in ``csrc/grid.cu`` — a
  counter-indexed Philox4x64-10 + Lemire restatement with a rejection
  fix-up, which the solver uses (``Restorer._grid``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import DataError

__all__ = ["SampleGrid", "axis_anchors", "regular_grid", "jitter_rng", "jittered_grid",
           "grid_draw_layout", "philox_key"]


@dataclass
class SampleGrid:
    positions: np.ndarray          # (n, 2) int64 (row, col)
    image_dims: tuple
    patch_side: int
    spacing: int
    mode: str
    offsets: np.ndarray | None = None
    global_shift: tuple = (0, 0)

    @property
    def n_patches(self) -> int:
        return int(self.positions.shape[0])

    @property
    def patch_dim(self) -> int:
        return self.patch_side * self.patch_side


def patch_side(patch_dim: int) -> int:
    side = math.isqrt(patch_dim)
    if side * side != patch_dim:
        raise DataError(f"patch_dim {patch_dim} is not a perfect square")
    return side


def axis_anchors(extent: int, side: int, spacing: int) -> np.ndarray:
    if extent < side:
        raise DataError(f"image extent {extent} smaller than patch side {side}")
    last = extent - side
    a = list(range(0, last + 1, spacing))
    if a[-1] != last:
        a.append(last)
    return np.asarray(a, dtype=np.int64)


def regular_grid(H: int, W: int, patch_dim: int, spacing: int) -> SampleGrid:
    side = patch_side(patch_dim)
    if not 1 <= spacing <= side:
        raise DataError(f"spacing must lie in [1, {side}], got {spacing}")
    r, c = np.meshgrid(axis_anchors(H, side, spacing), axis_anchors(W, side, spacing),
                       indexing="ij")
    return SampleGrid(np.stack([r.ravel(), c.ravel()], axis=1), (H, W), side, spacing, "regular")


def jitter_rng(seed: int, iteration: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & (2 ** 64 - 1), iteration]))


def philox_key(seed: int, iteration: int) -> tuple:
    """The two Philox key words numpy derives for jitter_rng(seed, iteration)
    (fed to the device generator so numpy's key-list conversion carries over)."""
    k = jitter_rng(seed, iteration).bit_generator.state["state"]["key"]
    return int(k[0]), int(k[1])


def jittered_grid(H: int, W: int, patch_dim: int, spacing: int,
                  rng: np.random.Generator) -> SampleGrid:
    base = regular_grid(H, W, patch_dim, spacing)
    side = base.patch_side
    half = (side - spacing) // 2
    if half == 0:
        return SampleGrid(base.positions, (H, W), side, spacing, "jittered",
                          offsets=np.zeros_like(base.positions))
    shift = rng.integers(0, spacing, size=2)
    band = shift % (2 * half + 1) - half
    jit = rng.integers(-half, half + 1, size=base.positions.shape)
    off = np.clip(band[None, :] + jit, -half, half)
    rows, cols = base.positions[:, 0], base.positions[:, 1]
    off[(rows == 0) | (rows == H - side), 0] = 0
    off[(cols == 0) | (cols == W - side), 1] = 0
    pos = base.positions + off
    np.clip(pos[:, 0], 0, H - side, out=pos[:, 0])
    np.clip(pos[:, 1], 0, W - side, out=pos[:, 1])
    return SampleGrid(pos, (H, W), side, spacing, "jittered", offsets=off,
                      global_shift=(int(shift[0]), int(shift[1])))


def grid_draw_layout(H: int, W: int, patch_dim: int, spacing: int) -> dict:
    """Parameters of the uint32 draw stream consumed by one jittered grid:
    ``n_shift`` global-shift draws over [0, spacing) then ``2n`` jitter draws
    over [-half, half], row-major (n, 2)."""
    side = patch_side(patch_dim)
    rows = axis_anchors(H, side, spacing)
    cols = axis_anchors(W, side, spacing)
    half = (side - spacing) // 2
    return {"side": side, "half": half, "n_rows": int(rows.size), "n_cols": int(cols.size),
            "n_shift": 0 if half == 0 or spacing == 1 else 2,
            "n_jitter": 0 if half == 0 else 2 * int(rows.size) * int(cols.size)}
