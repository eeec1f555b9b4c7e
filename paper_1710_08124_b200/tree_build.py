"""Offline search-tree construction: ``build_tree`` with its pairwise KL and
balanced-clustering local search on the device.

Restates `pkg/src/fepll/tree.py:68-227,315-380`:

* :func:`pairwise_symmetric_kl` (`tree.py:99-107`) — the K x K matrix of
  Tr(C_a^-1 C_b) is one FP64 matrix product over the P^2 flattened entries
  (``fepll_tree_kl``, csrc/tree_build.cu); the dense covariances and
  inverses are formed on the host exactly as `tree.py:72-87` does;
* :func:`balanced_cluster` (`tree.py:129-200`) — farthest-first medoid
  seeding and the greedy balanced fill on the host (O(K^2), the reference's
  numpy operations), the pairwise-swap local search (O(sweeps K^2), the
  reference's cost) on the device (``fepll_cluster_swap``), sequentially
  exact;
* :func:`collapse` / :func:`build_tree` (`tree.py:203-227,330-380`) — weight
  sums, weighted dense averages and the eigendecomposition on the host
  (LAPACK, as the reference) so the collapsed components, and the
  ``tree_write`` bytes, are the reference's.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import DataError
from .gmm import eigen_from_covariance, flatten_component
from .tree import GmmTree, TreeNode

__all__ = ["pairwise_symmetric_kl", "balanced_cluster", "collapse", "auto_level_sizes", "build_tree"]


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.DeviceError("no CUDA device: build_tree's KL and local search run on the GPU")
    return torch


def _cov_and_inv(comp):
    """`pkg/src/fepll/tree.py:72-87`"""
    P = comp.kept_basis.shape[0]
    r = comp.kept_basis.shape[1]
    ev = np.asarray(comp.kept_eigenvalues)
    spectrum_min = ev[-1] if r == P else min(comp.tail_value, ev[-1] if r else comp.tail_value)
    if spectrum_min <= 0:
        raise DataError("singular covariance: symmetric KL undefined")
    cov = comp.covariance()
    U = comp.kept_basis
    if r == P:
        inv = (U / ev) @ U.T
    else:
        inv = (U * (1.0 / ev - 1.0 / comp.tail_value)) @ U.T
        inv += np.eye(P) / comp.tail_value
    return cov, inv


def pairwise_symmetric_kl(components: Sequence) -> np.ndarray:
    """(K, K) symmetric KL, zero diagonal (`tree.py:99-107`), on the GPU."""
    torch = _torch()
    P = components[0].kept_basis.shape[0]
    if any(c.kept_basis.shape[0] != P for c in components):
        raise DataError("components have different patch_dim")
    pairs = [_cov_and_inv(c) for c in components]
    K = len(components)
    dev = torch.device("cuda")
    covs = torch.from_numpy(np.ascontiguousarray(np.stack([p[0] for p in pairs]))).to(dev)
    invs = torch.from_numpy(np.ascontiguousarray(np.stack([p[1] for p in pairs]))).to(dev)
    t = torch.empty((K, K), dtype=torch.float64, device=dev)
    kl = torch.empty((K, K), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    N.call("fepll_tree_kl", N.ptr(invs), N.ptr(covs), K, P, N.ptr(t), N.ptr(kl), st)
    return kl.cpu().numpy()


def _cluster_medoid(D: np.ndarray, members: list) -> int:
    sub = D[np.ix_(members, members)]
    return members[int(np.argmin(sub.sum(axis=1)))]


def balanced_cluster(components: Sequence, n_clusters: int, min_size: int, seed: int = 0,
                     sweeps: int = 200, divergences: np.ndarray | None = None) -> list:
    """`pkg/src/fepll/tree.py:129-200`: near-equal clusters with small
    within-cluster symmetric KL."""
    n = len(components)
    if n_clusters < 1:
        raise DataError("need at least one cluster")
    if n_clusters * min_size > n:
        raise DataError(f"cannot split {n} components into {n_clusters} "
                        f"clusters of at least {min_size}")
    if n // n_clusters < min_size:
        raise DataError(f"balanced clusters of {n} components into "
                        f"{n_clusters} groups violate min_size {min_size}")
    D = pairwise_symmetric_kl(components) if divergences is None else np.asarray(divergences, np.float64)
    rng = np.random.default_rng(seed)
    # farthest-first medoid seeding (tree.py:150-155)
    medoids = [int(rng.integers(n))]
    gap = D[medoids[0]].copy()
    while len(medoids) < n_clusters:
        gap[medoids] = -np.inf
        medoids.append(int(np.argmax(gap)))
        gap = np.minimum(gap, D[medoids[-1]])
    # greedy balanced fill (tree.py:157-167)
    clusters = [[m] for m in medoids]
    assigned = np.zeros(n, dtype=bool)
    assigned[medoids] = True
    while not assigned.all():
        sizes = [len(c) for c in clusters]
        target = int(np.argmin(sizes))
        medoid = _cluster_medoid(D, clusters[target])
        dist = D[medoid].copy()
        dist[assigned] = np.inf
        pick = int(np.argmin(dist))
        clusters[target].append(pick)
        assigned[pick] = True
    # pairwise-swap local search (tree.py:169-198) on the device
    cid = np.empty(n, dtype=np.int64)
    for l, members in enumerate(clusters):
        cid[members] = l
    rowsum = np.zeros((n, n_clusters))
    for l, members in enumerate(clusters):
        rowsum[:, l] = D[:, members].sum(axis=1)
    if sweeps > 0:
        torch = _torch()
        dev = torch.device("cuda")
        Dd = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
        cd = torch.from_numpy(cid).to(dev)
        rd = torch.from_numpy(rowsum).to(dev)
        done = torch.zeros(1, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        N.call("fepll_cluster_swap", N.ptr(Dd), n, n_clusters, N.ptr(cd), N.ptr(rd), int(sweeps),
               N.ptr(done), st)
        cid = cd.cpu().numpy()
    return [np.sort(np.where(cid == l)[0]) for l in range(n_clusters)]


def collapse(components: Sequence, partition: Sequence, rho: float) -> list:
    """`pkg/src/fepll/tree.py:203-227`."""
    seen = np.zeros(len(components), dtype=bool)
    out = []
    P = components[0].kept_basis.shape[0]
    for members in partition:
        members = np.asarray(members, dtype=np.int64)
        if members.size == 0:
            raise DataError("empty cluster in partition")
        if seen[members].any():
            raise DataError("partition reuses a component")
        seen[members] = True
        w = float(sum(components[k].weight for k in members))
        if w <= 0:
            raise DataError("zero-weight cluster")
        cov = np.zeros((P, P))
        for k in members:
            cov += components[k].weight * components[k].covariance()
        cov /= w
        out.append(flatten_component(w, eigen_from_covariance(cov), rho))
    if not seen.all():
        raise DataError("partition does not cover every component")
    return out


def auto_level_sizes(n_components: int) -> tuple:
    """`pkg/src/fepll/tree.py:315-327`: halving powers of two from the
    largest power that is at most K/2."""
    if n_components < 2:
        return ()
    top = 1
    while top * 2 <= n_components // 2:
        top *= 2
    sizes = []
    while top >= 1:
        sizes.append(top)
        top //= 2
    return tuple(sizes)


def build_tree(model, level_sizes: Sequence[int] | None = None, rho: float | None = None,
               seed: int = 0) -> GmmTree:
    """`pkg/src/fepll/tree.py:330-380`: collapse the mixture level by level
    into a search tree (leaf-adjacent clusters of >= 3 when feasible)."""
    model.validate()
    K = len(model.components)
    if level_sizes is None:
        level_sizes = auto_level_sizes(K)
    level_sizes = tuple(int(s) for s in level_sizes)
    if K == 1:
        if level_sizes:
            raise DataError("a single-component model admits only an empty level list")
        leaf = TreeNode(model.components[0], leaf_index=0, dense_cov=model.components[0].covariance())
        return GmmTree(leaf, (1,), model.patch_dim)
    if not level_sizes or level_sizes[-1] != 1:
        raise DataError("level_sizes must end at 1")
    if level_sizes[0] >= K:
        raise DataError(f"first level size {level_sizes[0]} must be below K={K}")
    if any(a <= b for a, b in zip(level_sizes, level_sizes[1:])):
        raise DataError("level_sizes must be strictly decreasing")
    if rho is None:
        rho = model.rho
    P = model.patch_dim
    nodes = [TreeNode(comp, leaf_index=k, dense_cov=comp.covariance())
             for k, comp in enumerate(model.components)]
    for depth_i, width in enumerate(level_sizes):
        comps = [node.component for node in nodes]
        min_size = 3 if depth_i == 0 and 3 * width <= len(nodes) else 2
        partition = balanced_cluster(comps, width, min_size, seed=seed + depth_i)
        nxt = []
        for members in partition:
            w = float(sum(comps[k].weight for k in members))
            dense = np.zeros((P, P))
            for k in members:
                dense += comps[k].weight * nodes[k].dense_cov
            dense /= w
            comp = flatten_component(w, eigen_from_covariance(dense), rho)
            nxt.append(TreeNode(comp, children=[nodes[k] for k in members], dense_cov=dense))
        nodes = nxt
    tree = GmmTree(nodes[0], (*reversed(level_sizes), K), P)
    tree.validate()
    return tree
