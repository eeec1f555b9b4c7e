"""Device-side degradation operator (C ABI ``fepll_op_*``).

Wraps one ``DegradationOperator`` (`pkg/src/fepll/operators.py:71-111`) as a
device plan: pixel maps / kernel taps / kernel DFT uploaded once, plus the
scratch of the cooperative CG and power-iteration kernels.  Host-side work
is limited to the closed-form ||A^T A||_F^2 of `operators.py:322-339` (a
sum over at most (2k-1)^2 kernel-autocorrelation lags) and drawing the power
iteration's start vector with the same generator call as the reference
(`default_rng(0).standard_normal`, `operators.py:304-305`).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import DataError

__all__ = ["DeviceOperator", "KIND_CODES", "frobenius_norm_sq_ata"]

KIND_CODES = {"identity": 0, "convolution": 1, "mask": 2, "gain": 3, "decimate": 4}


def _autocorr(kernel: np.ndarray) -> np.ndarray:
    """Linear autocorrelation a[d] = sum_q k[q] k[q + d], lags -(k-1)..(k-1)."""
    kh, kw = kernel.shape
    out = np.zeros((2 * kh - 1, 2 * kw - 1))
    for dr in range(-(kh - 1), kh):
        for dc in range(-(kw - 1), kw):
            a = kernel[max(0, -dr):kh - max(0, dr), max(0, -dc):kw - max(0, dc)]
            b = kernel[max(0, dr):kh - max(0, -dr), max(0, dc):kw - max(0, -dc)]
            out[dr + kh - 1, dc + kw - 1] = float(np.sum(a * b))
    return out


def frobenius_norm_sq_ata(A) -> float:
    """||A^T A||_F^2 in closed form (`pkg/src/fepll/operators.py:322-339`).

    For the kernel kinds, Parseval turns sum |khat|^4 into
    H W sum_d a[d]^2 over the kernel autocorrelation (exact while the
    autocorrelation support fits the image, checked here)."""
    H, W = (int(v) for v in A.input_dims)
    if A.kind == "identity":
        return float(H * W)
    if A.kind in ("mask", "gain"):
        pm = np.asarray(A.pixel_map, dtype=np.float64)
        d = (pm != 0).astype(np.float64) if A.kind == "mask" else pm * pm
        return float(np.sum(d ** 2))
    k = np.asarray(A.kernel, dtype=np.float64)
    kh, kw = k.shape
    if 2 * kh - 1 > H or 2 * kw - 1 > W:
        raise DataError("kernel too large relative to the image for the closed-form norm")
    auto = _autocorr(k)
    if A.kind == "convolution":
        return float(H * W * np.sum(auto ** 2))
    d = int(A.factor)
    lat = 0.0
    for i in range(2 * kh - 1):
        for j in range(2 * kw - 1):
            if (i - (kh - 1)) % d == 0 and (j - (kw - 1)) % d == 0:
                lat += auto[i, j] ** 2
    return float((H * W) / d ** 2 * lat)


def _cptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class DeviceOperator:
    def __init__(self, A):
        kind = A.kind
        if kind not in KIND_CODES:
            raise DataError(f"unknown operator kind {kind}")
        self.A = A
        self.kind = kind
        self.H, self.W = (int(v) for v in A.input_dims)
        self.Ho, self.Wo = (int(v) for v in A.output_dims)
        taps = None
        kh = kw = 0
        if kind in ("convolution", "decimate"):
            taps = np.ascontiguousarray(A.kernel, dtype=np.float64)
            kh, kw = taps.shape
        pm = None
        if kind in ("mask", "gain"):
            pm = np.asarray(A.pixel_map, dtype=np.float64)
            if kind == "mask":
                pm = (pm != 0).astype(np.float64)
            pm = np.ascontiguousarray(pm)
        h = C.c_void_p()
        N.call("fepll_op_create", KIND_CODES[kind], self.H, self.W, int(A.factor or 1),
               _cptr(taps), kh, kw, _cptr(pm), C.byref(h))
        self.handle = h

    def lambda_param(self, sigma: float) -> tuple:
        """(lambda, l2sq): `pkg/src/fepll/operators.py:342-355`."""
        v0 = np.ascontiguousarray(np.random.default_rng(0).standard_normal((self.H, self.W)))
        lam = C.c_double()
        l2 = C.c_double()
        N.call("fepll_op_lambda", self.handle, _cptr(v0), frobenius_norm_sq_ata(self.A),
               float(sigma), C.byref(lam), C.byref(l2))
        return float(lam.value), float(l2.value)

    def adjoint(self, y, out, stream):
        N.call("fepll_op_adjoint", self.handle, N.ptr(y), N.ptr(out), stream)

    def init(self, y, aty, sigma, lam, tol, maxit, x, info, stream):
        N.call("fepll_op_init", self.handle, N.ptr(y), N.ptr(aty), float(sigma), float(lam),
               float(tol), int(maxit), N.ptr(x), N.ptr(info), stream)

    def solve(self, rhs, xtilde, bs2, tol, maxit, x, info, status, stream):
        N.call("fepll_op_solve", self.handle, N.ptr(rhs), N.ptr(xtilde), float(bs2), float(tol),
               int(maxit), N.ptr(x), N.ptr(info), N.ptr(status), stream)

    def normal(self, x, shift, y, stream):
        N.call("fepll_op_normal", self.handle, N.ptr(x), float(shift), N.ptr(y), stream)

    def close(self):
        if getattr(self, "handle", None):
            N.lib().fepll_op_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
