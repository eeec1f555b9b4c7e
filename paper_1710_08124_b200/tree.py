"""Balanced Gaussian search tree: data model and the flattened device layout.

``TreeNode``/``GmmTree`` keep the reference field names
(`pkg/src/fepll/tree.py:234-312`) so reference trees are accepted as-is.
:func:`tree_topology` turns any such tree into the BFS arrays the CUDA walk
uses (children lists, leaf indices, depth), which is where the reference's
``tree_select`` starts as well (`pkg/src/fepll/tree.py:395-403`).

:func:`tree_from_partitions` rebuilds a tree from its level partitions by
the reference's collapse rule (`pkg/src/fepll/tree.py:359-378`): weights
add, dense covariances average with member weights in member order, then
eigendecompose and flatten at rho.  It lets the benchmark regenerate the
reference-built tree for the synthetic GMM on a box where the reference is
absent, from a few-KB partition fixture.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DataError
from .gmm import eigen_from_covariance, flatten_component

__all__ = ["TreeNode", "GmmTree", "TreeTopology", "tree_topology",
           "tree_from_partitions", "tree_partitions", "star_tree"]


@dataclass
class TreeNode:
    component: object
    children: list = field(default_factory=list)
    leaf_index: int | None = None
    dense_cov: np.ndarray | None = None

    @property
    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class GmmTree:
    root: TreeNode
    level_sizes: tuple
    patch_dim: int

    def bfs_nodes(self) -> list:
        order = [self.root]
        i = 0
        while i < len(order):
            order.extend(order[i].children)
            i += 1
        return order

    def bfs_components(self) -> list:
        return [n.component for n in self.bfs_nodes()]

    @property
    def n_leaves(self) -> int:
        return self.level_sizes[-1]

    @property
    def depth(self) -> int:
        return len(self.level_sizes) - 1

    def validate(self, tol: float = 1e-10) -> None:
        topo = tree_topology(self)
        for node in self.bfs_nodes():
            node.component.validate(tol)
            if not node.children:
                continue
            if len(node.children) < 2:
                raise DataError("internal node with fewer than 2 children")
            s = sum(c.component.weight for c in node.children)
            if abs(s - node.component.weight) > 1e-12:
                raise DataError("node weight differs from the sum of its children")
        if abs(self.root.component.weight - 1.0) > 1e-12:
            raise DataError("root weight differs from 1")
        widths = tuple(int(w) for w in np.bincount(topo.depth))
        if widths != tuple(self.level_sizes):
            raise DataError(f"recorded level sizes {self.level_sizes} != actual {widths}")


@dataclass
class TreeTopology:
    """BFS arrays: ``child_start[u]:child_start[u]+child_count[u]`` indexes
    ``child_list`` (BFS ids, in the node's stored child order)."""

    n_nodes: int
    child_start: np.ndarray
    child_count: np.ndarray
    child_list: np.ndarray
    leaf_index: np.ndarray  # -1 for internal nodes
    depth: np.ndarray
    parent: np.ndarray


def star_tree(model) -> GmmTree:
    """The exhaustive scan (gmm.py:371-391, select_exhaustive) as a one-level
    tree: the root's children are every component in index order, so the
    device descent takes the first minimum over all K scores — np.argmin's
    tie-break — and its path costs reproduce the no-tree counters of
    solver.py:154-157 (K evaluations, P + sum of score_flat_cost per patch).
    The root's own component is never scored."""
    comps = list(model.components)
    leaves = [TreeNode(component=c, leaf_index=k) for k, c in enumerate(comps)]
    return GmmTree(root=TreeNode(component=comps[0], children=leaves),
                   level_sizes=(1, len(comps)), patch_dim=int(model.patch_dim))


def tree_topology(tree) -> TreeTopology:
    nodes = tree.bfs_nodes()
    pos = {id(n): i for i, n in enumerate(nodes)}
    n = len(nodes)
    start = np.zeros(n, np.int32)
    count = np.zeros(n, np.int32)
    leaf = np.full(n, -1, np.int32)
    depth = np.zeros(n, np.int32)
    parent = np.full(n, -1, np.int32)
    flat = []
    for i, node in enumerate(nodes):
        start[i] = len(flat)
        count[i] = len(node.children)
        for c in node.children:
            j = pos[id(c)]
            flat.append(j)
            depth[j] = depth[i] + 1
            parent[j] = i
        if node.children:
            if node.leaf_index is not None:
                raise DataError("internal node carries a leaf_index")
        else:
            if node.leaf_index is None:
                raise DataError("leaf node without leaf_index")
            leaf[i] = int(node.leaf_index)
    leaves = np.sort(leaf[leaf >= 0])
    if not np.array_equal(leaves, np.arange(leaves.size)):
        raise DataError("leaf indices are not a permutation of 0..L-1")
    return TreeTopology(n, start, count, np.asarray(flat, np.int32), leaf, depth, parent)


def tree_partitions(tree) -> list:
    """Level partitions bottom-up: element ``d`` lists, for each node of the
    level above, the positions of its children within the level below (the
    inverse of :func:`tree_from_partitions`)."""
    nodes = tree.bfs_nodes()
    topo = tree_topology(tree)
    levels = [np.where(topo.depth == d)[0] for d in range(topo.depth.max() + 1)]
    # leaves are ordered by leaf index at the bottom level
    out = []
    below = {int(i): int(topo.leaf_index[i]) for i in levels[-1]}
    for d in range(len(levels) - 2, -1, -1):
        part = [[below[int(c)] for c in topo.child_list[topo.child_start[u]:
                                                         topo.child_start[u] + topo.child_count[u]]]
                for u in levels[d]]
        out.append(part)
        below = {int(u): k for k, u in enumerate(levels[d])}
    del nodes
    return out


def tree_from_partitions(model, partitions, rho: float | None = None) -> GmmTree:
    """Collapse ``model`` level by level along ``partitions`` (bottom-up, as
    returned by :func:`tree_partitions`)."""
    rho = model.rho if rho is None else rho
    P = model.patch_dim
    nodes = [TreeNode(c, leaf_index=k, dense_cov=c.covariance())
             for k, c in enumerate(model.components)]
    sizes = []
    for part in partitions:
        comps = [n.component for n in nodes]
        nxt = []
        for members in part:
            w = float(sum(comps[k].weight for k in members))
            dense = np.zeros((P, P))
            for k in members:
                dense += comps[k].weight * nodes[k].dense_cov
            dense /= w
            comp = flatten_component(w, eigen_from_covariance(dense), rho)
            nxt.append(TreeNode(comp, children=[nodes[k] for k in members], dense_cov=dense))
        nodes = nxt
        sizes.append(len(nodes))
    if len(nodes) != 1:
        raise DataError("partitions do not end at a single root")
    tree = GmmTree(nodes[0], (*reversed(sizes), model.n_components), P)
    tree.validate()
    return tree
