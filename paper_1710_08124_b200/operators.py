"""Degradation-operator interface (data model + constructors).

Same ``kind`` strings, fields and validation as the reference
(`pkg/src/fepll/operators.py:51-189`): identity | convolution | mask | gain |
decimate.  The arithmetic of ``apply``/``apply_adjoint``/the image solves
runs on the GPU (``csrc/operators.cu``); this module only describes the
operator and prepares its small host-side tables (kernel taps).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DataError

__all__ = [
    "CgConfig", "SolveInfo", "DegradationOperator", "identity_operator",
    "convolution_operator", "mask_operator", "gain_operator",
    "decimate_operator", "gaussian_kernel", "radial_gain_map",
]


@dataclass
class CgConfig:
    tolerance: float = 1e-6
    max_iterations: int = 200

    def validate(self) -> None:
        if self.tolerance <= 0:
            raise DataError("CG tolerance must be positive")
        if self.max_iterations < 1:
            raise DataError("CG needs at least one iteration")


@dataclass
class SolveInfo:
    method: str
    converged: bool
    iterations: int
    residual: float


_STRATEGY = {"identity": "pixel_diagonal", "mask": "pixel_diagonal",
             "gain": "pixel_diagonal", "convolution": "frequency_diagonal",
             "decimate": "iterative"}


@dataclass
class DegradationOperator:
    kind: str
    input_dims: tuple
    output_dims: tuple
    kernel: np.ndarray | None = None
    pixel_map: np.ndarray | None = None
    factor: int | None = None
    _kernel_ft: np.ndarray | None = field(default=None, repr=False)

    @property
    def solve_strategy(self) -> str:
        try:
            return _STRATEGY[self.kind]
        except KeyError:
            raise DataError(f"unknown operator kind {self.kind}") from None


def identity_operator(dims) -> DegradationOperator:
    return DegradationOperator("identity", tuple(dims), tuple(dims))


def convolution_operator(kernel, dims) -> DegradationOperator:
    kernel = np.asarray(kernel, dtype=np.float64)
    if kernel.ndim != 2 or kernel.shape[0] % 2 == 0 or kernel.shape[1] % 2 == 0:
        raise DataError(f"kernel must be 2-D with odd sides, got {kernel.shape}")
    if kernel.shape[0] > dims[0] or kernel.shape[1] > dims[1]:
        raise DataError("kernel larger than the image")
    return DegradationOperator("convolution", tuple(dims), tuple(dims), kernel=kernel)


def mask_operator(mask) -> DegradationOperator:
    binary = (np.asarray(mask) != 0).astype(np.float64)
    return DegradationOperator("mask", binary.shape, binary.shape, pixel_map=binary)


def gain_operator(gain) -> DegradationOperator:
    gain = np.asarray(gain, dtype=np.float64)
    if gain.min() < 0:
        raise DataError("gain map must be nonnegative")
    return DegradationOperator("gain", gain.shape, gain.shape, pixel_map=gain)


def gaussian_kernel(sigma: float, radius: int | None = None) -> np.ndarray:
    """Normalised separable Gaussian, side 2*radius+1, default radius
    ceil(3 sigma) (`pkg/src/fepll/operators.py:143-150`)."""
    if radius is None:
        radius = max(1, int(np.ceil(3.0 * sigma)))
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-0.5 * (t / sigma) ** 2)
    k = np.outer(g, g)
    return k / k.sum()


def decimate_operator(factor: int, input_dims, kernel=None) -> DegradationOperator:
    if factor < 2:
        raise DataError(f"decimation factor must be >= 2, got {factor}")
    H, W = input_dims
    if H % factor or W % factor:
        raise DataError(f"dims {tuple(input_dims)} not divisible by factor {factor}")
    if kernel is None:
        kernel = gaussian_kernel(0.5 * (factor - 1))
    kernel = np.asarray(kernel, dtype=np.float64)
    if kernel.shape[0] % 2 == 0 or kernel.shape[1] % 2 == 0:
        raise DataError("anti-alias kernel must have odd sides")
    return DegradationOperator("decimate", (H, W), (H // factor, W // factor),
                               kernel=kernel, factor=factor)


def radial_gain_map(dims, strength: float = 0.75) -> np.ndarray:
    H, W = dims
    r, c = np.meshgrid(np.arange(H) - (H - 1) / 2.0, np.arange(W) - (W - 1) / 2.0, indexing="ij")
    r2 = r ** 2 + c ** 2
    return 1.0 - strength * r2 / r2.max()
