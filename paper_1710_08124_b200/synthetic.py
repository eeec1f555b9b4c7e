"""Seeded synthetic inputs for the BASELINE configurations.

The paper's natural images and pretrained GMM are not available, so every
configuration of `BASELINE.json:configs` runs on:

* :func:`synthetic_image` — piecewise-smooth images: a random linear
  gradient, 20 random filled ellipses/rectangles with U[0,255]
  intensities, a Gaussian-smoothed N(0,1) texture rescaled to std 8,
  clipped to [0,255];
* :func:`synthetic_gmm` — K zero-mean components, Dirichlet(1) weights,
  random orthogonal eigenbases (QR with sign fix), spectrum
  lambda_i = (1e3 i^-1.5 + 0.1)/255^2 (8-bit^2 units rescaled to the [0,1]
  image scale the reference works in);
* :func:`baseline_tree` — the reference's balanced tree for that GMM,
  rebuilt from the committed partition fixture
  (``tests/golden/tree_partitions_P*.json``).

These generators are product-side input builders (bench + tests); they do
not depend on the reference package.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .gmm import Eigenbasis, GmmModel, component_from_eigen
from .operators import (convolution_operator, decimate_operator, gaussian_kernel,
                        identity_operator, mask_operator)

__all__ = ["synthetic_image", "synthetic_gmm", "baseline_tree", "BaselineCase",
           "baseline_case", "CONFIGS"]

_GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"


def synthetic_image(H: int, W: int, seed: int = 0, shapes: int = 20,
                    texture_std: float = 8.0) -> np.ndarray:
    """Piecewise-smooth test image on the 0..255 scale (float64)."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    r = np.arange(H, dtype=np.float64)[:, None] / max(H - 1, 1)
    c = np.arange(W, dtype=np.float64)[None, :] / max(W - 1, 1)
    g = rng.uniform(-1.0, 1.0, 2)
    img = rng.uniform(64.0, 192.0) + 96.0 * (g[0] * (r - 0.5) + g[1] * (c - 0.5))
    img = np.broadcast_to(img, (H, W)).copy()
    for _ in range(shapes):
        kind = rng.integers(0, 2)
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        ry, rx = rng.uniform(0.04, 0.25) * H, rng.uniform(0.04, 0.25) * W
        val = rng.uniform(0.0, 255.0)
        yy = np.arange(H)[:, None] - cy
        xx = np.arange(W)[None, :] - cx
        if kind == 0:
            inside = (yy / ry) ** 2 + (xx / rx) ** 2 <= 1.0
        else:
            inside = (np.abs(yy) <= ry) & (np.abs(xx) <= rx)
        img[inside] = val
    tex = gaussian_filter(rng.standard_normal((H, W)), 1.5)
    tex *= texture_std / tex.std()
    return np.clip(img + tex, 0.0, 255.0)


def synthetic_gmm(K: int = 200, patch_dim: int = 64, seed: int = 0, rho: float = 0.95) -> GmmModel:
    """Flat-tail model (rho) of the BASELINE synthetic spectrum."""
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.ones(K))
    w = w / w.sum()
    i = np.arange(1, patch_dim + 1, dtype=np.float64)
    lam = (1e3 * i ** -1.5 + 0.1) / 255.0 ** 2
    comps = []
    for k in range(K):
        Q, R = np.linalg.qr(rng.standard_normal((patch_dim, patch_dim)))
        Q = Q * np.sign(np.diag(R))[None, :]
        comps.append(component_from_eigen(float(w[k]), Eigenbasis(Q, lam.copy())))
    full = GmmModel(patch_dim, comps, 1.0)
    return full.flatten(rho) if rho < 1.0 else full


def baseline_tree(model: GmmModel, patch_dim: int | None = None):
    """Reference balanced tree of :func:`synthetic_gmm` (K=200, seed 0)."""
    from .tree import tree_from_partitions

    P = patch_dim or model.patch_dim
    path = _GOLDEN / f"tree_partitions_P{P}.json"
    parts = json.loads(path.read_text())["partitions"]
    return tree_from_partitions(model, parts)


@dataclass
class BaselineCase:
    name: str
    clean: np.ndarray       # [0,1] ground truth on the input grid
    y: np.ndarray           # [0,1] observation on the output grid
    A: object
    sigma8: float
    spacing: int
    patch_dim: int


def _noise(shape, sigma8: float, seed: int) -> np.ndarray:
    return sigma8 * np.random.default_rng(seed).standard_normal(shape)


def baseline_case(name: str, size: int | None = None, image_seed: int = 0,
                  noise_seed: int = 1) -> BaselineCase:
    """Inputs of one BASELINE configuration (optionally at a reduced size)."""
    spec = CONFIGS[name]
    H = W = size or spec["size"]
    img = synthetic_image(H, W, image_seed)
    s8 = spec["sigma"]
    kind = spec["op"]
    if kind == "identity":
        A = identity_operator((H, W))
        y = (img + _noise((H, W), s8, noise_seed)) / 255.0
    elif kind == "convolution":
        A = convolution_operator(gaussian_kernel(spec["blur_std"], spec["blur_radius"]), (H, W))
        blurred = _circular_conv(img, A.kernel)
        y = (blurred + _noise((H, W), s8, noise_seed)) / 255.0
    elif kind == "mask":
        mask = np.random.default_rng(noise_seed + 100).random((H, W)) < spec["keep"]
        A = mask_operator(mask)
        y = A.pixel_map * (img + _noise((H, W), s8, noise_seed)) / 255.0
    elif kind == "decimate":
        H = W = (H // spec["factor"]) * spec["factor"]
        img = img[:H, :W]
        A = decimate_operator(spec["factor"], (H, W),
                              gaussian_kernel(spec["blur_std"], spec["blur_radius"]))
        low = _circular_conv(img, A.kernel)[::spec["factor"], ::spec["factor"]]
        y = (low + _noise(low.shape, s8, noise_seed)) / 255.0
    else:
        raise ValueError(kind)
    return BaselineCase(name, img / 255.0, y, A, s8, spec["spacing"], spec["patch_dim"])


def _circular_conv(img: np.ndarray, kernel: np.ndarray) -> np.ndarray:
    """Periodic convolution with the kernel centred at the origin (the
    reference operator's forward model), done directly on the host to build
    observations."""
    kh, kw = kernel.shape
    out = np.zeros_like(img)
    for a in range(kh):
        for b in range(kw):
            out += kernel[a, b] * np.roll(img, (a - kh // 2, b - kw // 2), axis=(0, 1))
    return out


# BASELINE.json:configs, with the gotchas of SURVEY.md section 0.8 applied:
# [0,1] images with sigma on the 8-bit scale, 510x510 HR grid for x3 SR,
# default stride 6 where the config gives none, explicit kernel radii.
CONFIGS = {
    "cfg1": dict(size=256, op="identity", sigma=20.0, spacing=4, patch_dim=64),
    "cfg2": dict(size=512, op="identity", sigma=50.0, spacing=4, patch_dim=64),
    "cfg3": dict(size=512, op="convolution", sigma=2.0, spacing=2, patch_dim=64,
                 blur_std=1.6, blur_radius=4),
    "cfg4a": dict(size=512, op="mask", sigma=1.0, spacing=6, patch_dim=100, keep=0.5),
    "cfg4b": dict(size=510, op="decimate", sigma=1.0, spacing=6, patch_dim=100,
                  factor=3, blur_std=1.2, blur_radius=3),
    "cfg5": dict(size=1024, op="identity", sigma=25.0, spacing=4, patch_dim=64),
    "cfg5big": dict(size=8192, op="identity", sigma=25.0, spacing=4, patch_dim=64),
}
