"""Flat-tail GMM data model and the per-beta score constants (host plan).

The types keep the field names of the reference data model so either the
reference's objects or these can be handed to :func:`restore` (duck typing):

* ``FlatTailComponent`` — `pkg/src/fepll/gmm.py:96-155`
  (``weight``, ``kept_basis`` (P, r), ``kept_eigenvalues`` (r,), ``tail_value``)
* ``GmmModel`` — `pkg/src/fepll/gmm.py:191-251` (``patch_dim``, ``components``, ``rho``)

:func:`score_constants` restates the FP64 arithmetic of the reference's
``ScoreContext.__init__`` (`pkg/src/fepll/gmm.py:275-307`); the device plan
uploads its output once per HQS iteration.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import DataError

__all__ = [
    "Eigenbasis",
    "FlatTailComponent",
    "GmmModel",
    "eigen_from_covariance",
    "flatten_component",
    "component_from_eigen",
    "score_flat_cost",
    "wiener_flat_cost",
    "ScoreConstants",
    "score_constants",
]


@dataclass
class Eigenbasis:
    basis: np.ndarray        # (P, P) orthonormal columns
    eigenvalues: np.ndarray  # (P,) non-increasing, >= 0


@dataclass
class FlatTailComponent:
    weight: float
    kept_basis: np.ndarray        # (P, rank)
    kept_eigenvalues: np.ndarray  # (rank,)
    tail_value: float

    @property
    def patch_dim(self) -> int:
        return int(self.kept_basis.shape[0])

    @property
    def rank(self) -> int:
        return int(self.kept_basis.shape[1])

    @property
    def tail_dim(self) -> int:
        return self.patch_dim - self.rank

    def covariance(self) -> np.ndarray:
        """U diag(s - t) U^T + t I (`pkg/src/fepll/gmm.py:132-138`)."""
        U = self.kept_basis
        cov = (U * (self.kept_eigenvalues - self.tail_value)) @ U.T
        cov += self.tail_value * np.eye(self.patch_dim)
        return cov

    def validate(self, tol: float = 1e-10) -> None:
        if not self.weight > 0:
            raise DataError(f"component weight must be positive, got {self.weight}")
        if self.tail_value < 0:
            raise DataError(f"negative tail value {self.tail_value}")
        if np.shape(self.kept_eigenvalues) != (self.rank,):
            raise DataError("kept eigenvalue count does not match basis rank")
        if self.rank:
            g = self.kept_basis.T @ self.kept_basis
            if np.abs(g - np.eye(self.rank)).max() > tol:
                raise DataError("kept basis not orthonormal")
            ev = np.asarray(self.kept_eigenvalues)
            if np.any(np.diff(ev) > 0) or ev[-1] < 0:
                raise DataError("kept eigenvalues must be non-increasing and nonnegative")
            if self.rank < self.patch_dim and ev[-1] < self.tail_value - tol:
                raise DataError("flat tail exceeds the smallest kept eigenvalue")


@dataclass
class GmmModel:
    patch_dim: int
    components: list
    rho: float = 1.0

    @property
    def n_components(self) -> int:
        return len(self.components)

    @property
    def weights(self) -> np.ndarray:
        return np.array([c.weight for c in self.components], dtype=np.float64)

    @property
    def ranks(self) -> np.ndarray:
        return np.array([c.kept_basis.shape[1] for c in self.components])

    @property
    def is_full_rank(self) -> bool:
        return bool(np.all(self.ranks == self.patch_dim))

    def validate(self, tol: float = 1e-10) -> None:
        if self.n_components == 0:
            raise DataError("model must contain at least one component")
        if not 0.0 < self.rho <= 1.0:
            raise DataError(f"rho must lie in (0, 1], got {self.rho}")
        for k, c in enumerate(self.components):
            if c.kept_basis.shape[0] != self.patch_dim:
                raise DataError(f"component {k} patch_dim mismatch")
            c.validate(tol)
        s = self.weights.sum()
        if abs(s - 1.0) > 1e-12:
            raise DataError(f"component weights sum to {s!r}, expected 1")

    def flatten(self, rho: float) -> "GmmModel":
        if not self.is_full_rank:
            raise DataError("model is already flat-tail compressed")
        comps = [flatten_component(c.weight, Eigenbasis(c.kept_basis, c.kept_eigenvalues), rho)
                 for c in self.components]
        return GmmModel(self.patch_dim, comps, rho)


def eigen_from_covariance(cov: np.ndarray) -> Eigenbasis:
    """Descending eigenpairs of a symmetric PSD matrix, eigenvalues clamped
    at 0 (`pkg/src/fepll/gmm.py:75-93`)."""
    cov = np.asarray(cov, dtype=np.float64)
    if cov.ndim != 2 or cov.shape[0] != cov.shape[1]:
        raise DataError(f"covariance must be square, got {cov.shape}")
    if np.abs(cov - cov.T).max() > 1e-10:
        raise DataError("covariance not symmetric")
    vals, vecs = np.linalg.eigh(cov)
    if vals[0] < -1e-6:
        raise DataError("eigenvalue below -1e-6: not a covariance")
    return Eigenbasis(np.ascontiguousarray(vecs[:, ::-1]), np.clip(vals[::-1], 0.0, None))


def component_from_eigen(weight: float, eig: Eigenbasis) -> FlatTailComponent:
    return FlatTailComponent(weight, eig.basis.copy(), eig.eigenvalues.copy(), 0.0)


def flatten_component(weight: float, eig: Eigenbasis, rho: float) -> FlatTailComponent:
    """Keep the smallest rank explaining ``rho`` of the trace; the rest
    becomes a flat tail at their mean (`pkg/src/fepll/gmm.py:163-188`)."""
    if not 0.0 < rho <= 1.0:
        raise DataError(f"rho must lie in (0, 1], got {rho}")
    vals = eig.eigenvalues
    P = vals.shape[0]
    cum = np.cumsum(vals)
    total = cum[-1] if P else 0.0
    if total <= 0.0:
        return FlatTailComponent(weight, eig.basis[:, :0].copy(), vals[:0].copy(), 0.0)
    rank = P if rho == 1.0 else min(int(np.searchsorted(cum, rho * total, side="left")) + 1, P)
    tail = float(vals[rank:].mean()) if rank < P else 0.0
    return FlatTailComponent(weight, np.ascontiguousarray(eig.basis[:, :rank]),
                             vals[:rank].copy(), tail)


def score_flat_cost(rank: int, patch_dim: int) -> int:
    """Multiplies per flat score evaluation (`pkg/src/fepll/gmm.py:254-257`)."""
    return rank * patch_dim + 2 * rank + 1


def wiener_flat_cost(rank: int, patch_dim: int) -> int:
    """Multiplies per flat Wiener estimate (`pkg/src/fepll/gmm.py:260-263`)."""
    return rank * patch_dim + rank + patch_dim


@dataclass
class ScoreConstants:
    """FP64 per-component constants at one beta, component-major.

    ``sq_weight[k]`` = 1/nu - 1/nu_tail and ``shrink[k]`` = gamma - gamma_tail
    are (rank_k,) vectors; ``const[k]`` = iota + tail_dim*log(nu_tail) +
    sum(log nu); ``nu_tail``, its reciprocal, and ``gamma_tail``.
    """

    beta: float
    const: np.ndarray
    nu_tail: np.ndarray
    inv_nu_tail: np.ndarray
    gamma_tail: np.ndarray
    sq_weight: list
    shrink: list


def score_constants(components: Sequence, beta: float) -> ScoreConstants:
    """Restates `pkg/src/fepll/gmm.py:275-307` operation for operation."""
    if not beta > 0:
        raise DataError(f"beta must be positive, got {beta}")
    if len(components) == 0:
        raise DataError("score context needs at least one component")
    inv_beta = 1.0 / beta
    K = len(components)
    const = np.empty(K)
    nu_tails = np.empty(K)
    inv_nu_tail = np.empty(K)
    gamma_tail = np.empty(K)
    sq_w, shrink = [], []
    for k, c in enumerate(components):
        ev = np.asarray(c.kept_eigenvalues, dtype=np.float64)
        nu = ev + inv_beta
        nu_tail = c.tail_value + inv_beta
        if nu_tail <= 0 or (nu.size and nu.min() <= 0):
            raise DataError("nonpositive nu; spectrum or beta invalid")
        gamma = ev / nu
        g_tail = c.tail_value / nu_tail
        iota = -2.0 * math.log(c.weight)
        tail_dim = c.kept_basis.shape[0] - c.kept_basis.shape[1]
        sq_w.append(1.0 / nu - 1.0 / nu_tail)
        const[k] = iota + tail_dim * math.log(nu_tail) + np.log(nu).sum()
        shrink.append(gamma - g_tail)
        nu_tails[k] = nu_tail
        inv_nu_tail[k] = 1.0 / nu_tail
        gamma_tail[k] = g_tail
    return ScoreConstants(float(beta), const, nu_tails, inv_nu_tail, gamma_tail, sq_w, shrink)
