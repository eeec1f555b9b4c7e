"""FEPLLGM1 / FEPLLTR1 readers and writers (host ingestion).

Byte layouts follow the reference formats so the same files feed the CPU
oracle and this package (`pkg/src/fepll/model_io.py:1-20`,
`pkg/src/fepll/tree.py:15-26`):

model:  b"FEPLLGM1", K u32, P u32, rho f64, then K component payloads
tree:   b"FEPLLTR1", nodes u32, P u32, then per BFS node a component
        payload, child_count u32, children u32[], leaf_index i32
payload: weight f64, rank u32, tail f64, eigenvalues f64[rank],
         basis f64[P*rank] column-major
"""

from __future__ import annotations

import io
import struct
from pathlib import Path

import numpy as np

from .errors import DataError
from .gmm import FlatTailComponent, GmmModel

__all__ = ["MODEL_MAGIC", "TREE_MAGIC", "model_read", "model_write",
           "tree_read", "tree_write"]

MODEL_MAGIC = b"FEPLLGM1"
TREE_MAGIC = b"FEPLLTR1"
_HEAD = struct.Struct("<dId")


def _take(buf: io.BufferedIOBase, n: int, what: str) -> bytes:
    b = buf.read(n)
    if len(b) != n:
        raise DataError(f"truncated file while reading {what}")
    return b


def _put_component(fh, comp) -> None:
    basis = np.asarray(comp.kept_basis, dtype="<f8")
    fh.write(_HEAD.pack(float(comp.weight), basis.shape[1], float(comp.tail_value)))
    fh.write(np.asarray(comp.kept_eigenvalues, dtype="<f8").tobytes())
    fh.write(basis.tobytes(order="F"))


def _get_component(fh, P: int, idx: int) -> FlatTailComponent:
    weight, rank, tail = _HEAD.unpack(_take(fh, _HEAD.size, f"component {idx}"))
    if rank > P:
        raise DataError(f"component {idx}: rank {rank} exceeds patch_dim {P}")
    ev = np.frombuffer(_take(fh, 8 * rank, f"component {idx} eigenvalues"), "<f8").astype(np.float64)
    raw = np.frombuffer(_take(fh, 8 * rank * P, f"component {idx} basis"), "<f8")
    basis = np.array(raw.reshape((rank, P)).T, dtype=np.float64, order="C")
    return FlatTailComponent(weight, basis, ev, tail)


def model_write(model, path) -> None:
    with open(path, "wb") as fh:
        fh.write(MODEL_MAGIC)
        fh.write(struct.pack("<IId", len(model.components), int(model.patch_dim), float(model.rho)))
        for c in model.components:
            _put_component(fh, c)


def model_read(path) -> GmmModel:
    with open(path, "rb") as fh:
        if fh.read(8) != MODEL_MAGIC:
            raise DataError(f"{path}: not a FEPLLGM1 model file")
        K, P, rho = struct.unpack("<IId", _take(fh, 16, "header"))
        if K == 0 or P == 0:
            raise DataError(f"{path}: empty model header")
        comps = [_get_component(fh, P, k) for k in range(K)]
        if fh.read(1):
            raise DataError(f"{path}: trailing bytes")
    m = GmmModel(P, comps, rho)
    m.validate()
    return m


def tree_write(tree, path) -> None:
    nodes = tree.bfs_nodes()
    pos = {id(n): i for i, n in enumerate(nodes)}
    with open(path, "wb") as fh:
        fh.write(TREE_MAGIC)
        fh.write(struct.pack("<II", len(nodes), int(tree.patch_dim)))
        for n in nodes:
            _put_component(fh, n.component)
            kids = [pos[id(c)] for c in n.children]
            fh.write(struct.pack("<I", len(kids)))
            if kids:
                fh.write(struct.pack(f"<{len(kids)}I", *kids))
            fh.write(struct.pack("<i", -1 if n.leaf_index is None else int(n.leaf_index)))


def tree_read(path):
    from .tree import GmmTree, TreeNode

    with open(path, "rb") as fh:
        if fh.read(8) != TREE_MAGIC:
            raise DataError(f"{path}: not a FEPLLTR1 tree file")
        count, P = struct.unpack("<II", _take(fh, 8, "header"))
        if count == 0 or P == 0:
            raise DataError(f"{path}: empty tree header")
        nodes, kids_of = [], []
        for i in range(count):
            comp = _get_component(fh, P, i)
            (nk,) = struct.unpack("<I", _take(fh, 4, f"node {i} child count"))
            kids = list(struct.unpack(f"<{nk}I", _take(fh, 4 * nk, f"node {i} children"))) if nk else []
            (leaf,) = struct.unpack("<i", _take(fh, 4, f"node {i} leaf index"))
            nodes.append(TreeNode(comp, leaf_index=None if leaf < 0 else leaf))
            kids_of.append(kids)
        if fh.read(1):
            raise DataError(f"{path}: trailing bytes")
    refs = np.zeros(count, dtype=int)
    depth = np.zeros(count, dtype=int)
    for i, kids in enumerate(kids_of):
        for j in kids:
            if j <= i or j >= count:
                raise DataError(f"{path}: node {i} references invalid child {j}")
            refs[j] += 1
            depth[j] = depth[i] + 1
        nodes[i].children = [nodes[j] for j in kids]
    if refs[0] != 0 or np.any(refs[1:] != 1):
        raise DataError(f"{path}: nodes must form a single rooted tree")
    widths = tuple(int((depth == d).sum()) for d in range(depth.max() + 1))
    tree = GmmTree(nodes[0], widths, P)
    tree.validate()
    return tree
