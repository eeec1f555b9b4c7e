"""Host packing of a GmmModel + GmmTree into the device plan.

Layout in HBM (all FP64 unless stated):

* group block of internal node u (BFS id): the kept bases of its children
  side by side, P x width_u row-major (``grp_basis[grp_off64[u]:]``) — one
  pass over z computes every child's projection;
* ``grp_sqw[t]``: per group column, sq_weight = 1/nu - 1/nu_tail of the
  child owning the column at beta_t; ``node_const[t]``/``node_nu_tail[t]``
  per node as a child (gmm.py:291-307 via :func:`gmm.score_constants`);
* model block of component k: P x r_k row-major for the Wiener step, with
  ``model_shrink[t]`` = gamma - gamma_tail per column and
  ``model_gamma_tail[t]``;
* tcgen05 operand images (FP32, TF32 hi/lo split, K-major 128B-swizzled,
  each child padded to 16 columns) and their FP32 column weights: see
  ``tc_images``.

The whole beta schedule is packed once, so nothing is uploaded inside the
restoration loop.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import DataError
from .gmm import score_constants
from .tree import tree_topology

__all__ = ["DevicePlan", "pack_plan", "tc_images"]


def _c(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def tf32_split(a: np.ndarray):
    """FP32 value -> (hi, lo) with hi rounded to TF32 (10-bit mantissa, RNE)
    and lo = fp32(a - hi); hi + lo carries ~22 significant bits."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    rounded = ((bits + 0xFFF + ((bits >> 13) & 1)) & 0xFFFFE000).astype(np.uint32)
    hi = rounded.view(np.float32)
    lo = (a.astype(np.float64) - hi.astype(np.float64)).astype(np.float32)
    return hi, lo


def bf16_rne(a: np.ndarray) -> np.ndarray:
    """FP32 -> bfloat16 bit patterns (uint16), round to nearest even."""
    bits = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16).astype(np.uint16)


def bf16_cross_image(hi: np.ndarray, lo: np.ndarray) -> np.ndarray:
    """B operand of the bf16 cross pass: rows x (2 Ppad) bfloat16 K-major
    [bf16(lo) | bf16(hi)] (it meets A = [bf16(z_hi) | bf16(z_lo)], so the
    pass adds z_hi . b_lo + z_lo . b_hi), packed two per 32-bit word (lower K
    in the low half) and 128B-swizzled like the FP32 images — same bytes."""
    rows, Ppad = hi.shape
    x = np.concatenate([bf16_rne(lo), bf16_rne(hi)], axis=1).astype(np.uint32)  # (rows, 2 Ppad)
    words = (x[:, 0::2] | (x[:, 1::2] << 16)).astype(np.uint32)                   # (rows, Ppad)
    return swizzle128_kmajor(words.view(np.float32))


def swizzle128_kmajor(mat: np.ndarray) -> np.ndarray:
    """Rows x 64-float (256 B) K-major matrix -> the byte image tcgen05
    expects for SWIZZLE_128B K-major operands: K split in 32-float (128 B)
    atoms, each atom an [rows/8][8 rows][128 B] stack, 16-byte chunks XORed
    with (row % 8).  ``mat`` is (rows, K) with rows % 8 == 0, K % 32 == 0."""
    rows, K = mat.shape
    assert rows % 8 == 0 and K % 32 == 0
    out = np.zeros(rows * K, dtype=np.float32)
    katoms = K // 32
    for ka in range(katoms):
        blk = mat[:, ka * 32:(ka + 1) * 32]            # (rows, 32)
        chunks = blk.reshape(rows, 8, 4)               # 8 chunks of 16 B
        r = np.arange(rows)
        dst = np.empty_like(chunks)
        for ch in range(8):
            dst[r, ch ^ (r % 8), :] = chunks[:, ch, :]
        base = ka * rows * 32
        out[base:base + rows * 32] = dst.reshape(-1)
    return out


def tc_images(topo, comps, P: int, sqw_per_node: list):
    """Operands of the tcgen05 scorer, one set per beta_t.

    For internal node u and iteration t the B image is the group matrix with
    every column scaled by sqrt(-w_t) (w_t = sq_weight at beta_t, <= 0 for a
    flat-tail model: kept eigenvalues >= the tail value), transposed to
    (npad_u, P_pad) K-major — child v occupying rows
    [tc_child_col[v], tc_child_col[v] + r_v), every child padded to a multiple
    of 16 rows so each child starts on a 16-column TMEM chunk — then TF32
    hi/lo split and 128B-swizzled (``tc_x``: the bf16 [lo | hi] image of the
    mixed-precision scorer, select_ws2.cu).  The scorer's epilogue then needs only
    -sum_j c'_j^2 per child (c' = z . B'), no per-column weights.  Images are
    laid out [T][nodes]; ``tc_off`` is the offset within one iteration's
    block.  ``sqw_per_node[t][v]`` (FP64 vectors) also become the FP32
    per-column weights ``tc_w`` (0 on padding) that the error bound's
    ||w_c|| is taken from.  Returns None if some weight is positive."""
    Ppad = ((P + 31) // 32) * 32
    n = topo.n_nodes
    tc_off = np.zeros(n, np.int64)
    tc_npad = np.zeros(n, np.int32)
    tc_child_col = np.zeros(n, np.int32)
    tc_w_off = np.zeros(n, np.int32)
    cur = 0
    wcols = 0
    groups = []
    for u in range(n):
        nk = topo.child_count[u]
        if nk == 0:
            continue
        kids = topo.child_list[topo.child_start[u]:topo.child_start[u] + nk]
        col = 0
        for v in kids:
            tc_child_col[v] = col
            col += ((comps[v].kept_basis.shape[1] + 15) // 16) * 16
        npad = max(col, 16)
        tc_off[u] = cur
        tc_npad[u] = npad
        tc_w_off[u] = wcols
        cur += npad * Ppad
        wcols += npad
        groups.append((u, kids))
    T = len(sqw_per_node)
    for t in range(T):
        for u, kids in groups:
            for v in kids:
                if np.any(np.asarray(sqw_per_node[t][v]) > 0):
                    return None
    his, los, xs = [], [], []
    for t in range(T):
        for u, kids in groups:
            Bt = np.zeros((tc_npad[u], Ppad), dtype=np.float64)
            for v in kids:
                r = comps[v].kept_basis.shape[1]
                scale = np.sqrt(-np.asarray(sqw_per_node[t][v], dtype=np.float64))
                Bt[tc_child_col[v]:tc_child_col[v] + r, :P] = (np.asarray(comps[v].kept_basis)
                                                               * scale[None, :]).T
            hi, lo = tf32_split(Bt.astype(np.float32))
            hi = hi.reshape(tc_npad[u], Ppad)
            lo = lo.reshape(tc_npad[u], Ppad)
            his.append(swizzle128_kmajor(hi))
            los.append(swizzle128_kmajor(lo))
            xs.append(bf16_cross_image(hi, lo))
    tc_w = np.zeros((T, max(wcols, 1)), np.float32)
    for t in range(T):
        for u, kids in groups:
            for v in kids:
                a0 = tc_w_off[u] + tc_child_col[v]
                w = sqw_per_node[t][v]
                tc_w[t, a0:a0 + w.size] = w.astype(np.float32)
    return dict(tc_hi=np.concatenate(his) if his else np.zeros(0, np.float32),
                tc_lo=np.concatenate(los) if los else np.zeros(0, np.float32),
                tc_x=np.concatenate(xs) if xs else np.zeros(0, np.float32),
                tc_off=tc_off, tc_npad=tc_npad, tc_child_col=tc_child_col,
                tc_w=tc_w, tc_w_off=tc_w_off, tc_w_cols=max(wcols, 1), tc_tstride=cur)


def pack_plan(model, tree, betas, with_tc: bool = True) -> dict:
    """All host arrays of the plan descriptor (numpy, contiguous)."""
    P = int(model.patch_dim)
    K = len(model.components)
    topo = tree_topology(tree)
    nodes = tree.bfs_nodes()
    n = topo.n_nodes
    comps = [nd.component for nd in nodes]
    rank = np.array([c.kept_basis.shape[1] for c in comps], np.int32)
    if tree.patch_dim != P:
        raise DataError("tree patch_dim differs from the model's")
    grp_width = np.zeros(n, np.int32)
    grp_col_off = np.zeros(n, np.int32)
    child_col_off = np.zeros(n, np.int32)
    grp_off64 = np.zeros(n, np.int64)
    blocks, bl = [], {}
    col = 0
    el = 0
    for u in range(n):
        nk = topo.child_count[u]
        if nk == 0:
            continue
        kids = topo.child_list[topo.child_start[u]:topo.child_start[u] + nk]
        w = 0
        for v in kids:
            child_col_off[v] = w
            w += rank[v]
        G = np.concatenate([np.asarray(comps[v].kept_basis, np.float64) for v in kids], axis=1)
        grp_width[u] = w
        grp_col_off[u] = col
        grp_off64[u] = el
        col += w
        el += P * w
        blocks.append(np.ascontiguousarray(G).reshape(-1))
        bl[u] = G
    grp_basis = np.concatenate(blocks) if blocks else np.zeros(1)
    T = len(betas)
    node_const = np.zeros((T, n))
    node_nu_tail = np.zeros((T, n))
    grp_sqw = np.zeros((T, max(col, 1)))
    mrank = np.array([c.kept_basis.shape[1] for c in model.components], np.int32)
    mcol = np.concatenate([[0], np.cumsum(mrank)[:-1]]).astype(np.int32)
    moff = (mcol.astype(np.int64) * P)
    mbasis = np.concatenate([np.ascontiguousarray(np.asarray(c.kept_basis, np.float64)).reshape(-1)
                             for c in model.components])
    mcols = int(mrank.sum())
    shrink = np.zeros((T, max(mcols, 1)))
    gtail = np.zeros((T, K))
    sqw_nodes = []
    for t, beta in enumerate(betas):
        sc = score_constants(comps, float(beta))
        sqw_nodes.append(sc.sq_weight)
        node_const[t] = sc.const
        node_nu_tail[t] = sc.nu_tail
        for u in bl:
            kids = topo.child_list[topo.child_start[u]:topo.child_start[u] + topo.child_count[u]]
            for v in kids:
                a = grp_col_off[u] + child_col_off[v]
                grp_sqw[t, a:a + rank[v]] = sc.sq_weight[v]
        mc = score_constants(model.components, float(beta))
        for k in range(K):
            shrink[t, mcol[k]:mcol[k] + mrank[k]] = mc.shrink[k]
        gtail[t] = mc.gamma_tail
    out = dict(P=P, n=n, K=K, T=T, topo=topo, rank=rank, grp_width=grp_width,
               grp_col_off=grp_col_off, child_col_off=child_col_off, grp_off64=grp_off64,
               grp_basis=grp_basis, grp_cols=col, node_const=node_const,
               node_nu_tail=node_nu_tail, grp_sqw=grp_sqw, mrank=mrank, mcol=mcol, moff=moff,
               mbasis=mbasis, mcols=mcols, shrink=shrink, gtail=gtail, blocks=bl)
    if with_tc:
        tc = tc_images(topo, comps, P, sqw_nodes)
        if tc is not None:  # (a positive sq_weight leaves tensor mode unavailable)
            out.update(tc)
    # per-leaf path costs for the reference's counters (tree.py:413-427)
    out["path_evals"], out["path_mults"] = _path_costs(topo, rank, P)
    return out


def _path_costs(topo, rank, P):
    """evals / mults accumulated on the unique root->leaf path of each leaf
    (tree.py:413-427): every visited internal node adds |children| and the
    score_flat_cost of each child."""
    n = topo.n_nodes
    ev = np.zeros(n, np.int64)
    mu = np.zeros(n, np.int64)
    mu[0] = P
    for u in range(n):
        nk = topo.child_count[u]
        if nk == 0:
            continue
        kids = topo.child_list[topo.child_start[u]:topo.child_start[u] + nk]
        cost = int(sum(int(rank[v]) * P + 2 * int(rank[v]) + 1 for v in kids))
        for v in kids:
            ev[v] = ev[u] + nk
            mu[v] = mu[u] + cost
    K = int(topo.leaf_index.max()) + 1
    pe = np.zeros(K, np.int64)
    pm = np.zeros(K, np.int64)
    for u in range(n):
        if topo.leaf_index[u] >= 0:
            pe[topo.leaf_index[u]] = ev[u]
            pm[topo.leaf_index[u]] = mu[u]
    return pe, pm


class DevicePlan:
    """Owns the C plan handle for one (model, tree, beta schedule)."""

    def __init__(self, model, tree, betas, with_tc: bool = True):
        self.host = h = pack_plan(model, tree, betas, with_tc)
        topo = h["topo"]
        keep = {}

        def arr(name, a, dt):
            keep[name] = np.ascontiguousarray(a, dtype=dt)
            return keep[name]

        d = N.PlanDesc()
        d.patch_dim, d.n_nodes, d.n_components, d.iterations = h["P"], h["n"], h["K"], h["T"]
        d.child_start = _c(arr("cs", topo.child_start, np.int32), C.c_int32)
        d.child_count = _c(arr("cc", topo.child_count, np.int32), C.c_int32)
        d.child_list = _c(arr("cl", topo.child_list if topo.child_list.size else [0], np.int32), C.c_int32)
        d.leaf_index = _c(arr("li", topo.leaf_index, np.int32), C.c_int32)
        d.depth = _c(arr("de", topo.depth, np.int32), C.c_int32)
        d.node_rank = _c(arr("nr", h["rank"], np.int32), C.c_int32)
        d.grp_width = _c(arr("gw", h["grp_width"], np.int32), C.c_int32)
        d.grp_col_off = _c(arr("gc", h["grp_col_off"], np.int32), C.c_int32)
        d.child_col_off = _c(arr("cco", h["child_col_off"], np.int32), C.c_int32)
        d.grp_off64 = _c(arr("go", h["grp_off64"], np.int64), C.c_int64)
        d.grp_basis = _c(arr("gb", h["grp_basis"], np.float64), C.c_double)
        d.grp_basis_len = keep["gb"].size
        d.grp_cols_total = max(h["grp_cols"], 1)
        d.node_const = _c(arr("ncst", h["node_const"], np.float64), C.c_double)
        d.node_nu_tail = _c(arr("nnt", h["node_nu_tail"], np.float64), C.c_double)
        d.grp_sqw = _c(arr("sqw", h["grp_sqw"], np.float64), C.c_double)
        d.model_rank = _c(arr("mr", h["mrank"], np.int32), C.c_int32)
        d.model_col_off = _c(arr("mc", h["mcol"], np.int32), C.c_int32)
        d.model_off64 = _c(arr("mo", h["moff"], np.int64), C.c_int64)
        d.model_basis = _c(arr("mb", h["mbasis"], np.float64), C.c_double)
        d.model_basis_len = keep["mb"].size
        d.model_cols_total = max(h["mcols"], 1)
        d.model_shrink = _c(arr("ms", h["shrink"], np.float64), C.c_double)
        d.model_gamma_tail = _c(arr("mg", h["gtail"], np.float64), C.c_double)
        self.has_tc = bool(with_tc and "tc_hi" in h and h["tc_hi"].size)
        if self.has_tc:
            d.grp_tc_hi = _c(arr("th", h["tc_hi"], np.float32), C.c_float)
            d.grp_tc_lo = _c(arr("tl", h["tc_lo"], np.float32), C.c_float)
            d.grp_tc_len = keep["th"].size
            d.grp_tc_off = _c(arr("to", h["tc_off"], np.int64), C.c_int64)
            d.grp_tc_npad = _c(arr("tn", h["tc_npad"], np.int32), C.c_int32)
            d.grp_tc_child_col = _c(arr("tcc", h["tc_child_col"], np.int32), C.c_int32)
            d.grp_tc_w = _c(arr("tw", h["tc_w"], np.float32), C.c_float)
            d.grp_tc_w_off = _c(arr("two", h["tc_w_off"], np.int32), C.c_int32)
            d.grp_tc_w_cols = int(h["tc_w_cols"])
            d.grp_tc_x = _c(arr("tx", h["tc_x"], np.float32), C.c_float)
        handle = C.c_void_p()
        N.call("fepll_plan_create", C.byref(d), C.byref(handle))
        self.handle = handle
        self.P, self.K, self.T = h["P"], h["K"], h["T"]
        self.path_evals = h["path_evals"]
        self.path_mults = h["path_mults"]
        self.reserved = 0

    OPTIONS = ("select_variant", "seg_sq", "wiener_pair", "wiener_rw", "wiener_xw", "wiener_add_dc",
               "l2_prefetch", "rescore_by_node", "aggregate_variant", "wiener_split", "wiener_tc", "wiener_ws", "pdl",
               "defer", "defer_test")

    def set_option(self, name: str, value: int) -> None:
        """Per-plan kernel choice (include/fepll_b200.h fepll_plan_set_option)."""
        N.call("fepll_plan_set_option", self.handle, name.encode(), int(value))

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        N.call("fepll_plan_get_option", self.handle, name.encode(), C.byref(v))
        return int(v.value)

    def reserve(self, n_patches: int) -> None:
        if n_patches > self.reserved:
            N.call("fepll_plan_reserve", self.handle, int(n_patches))
            self.reserved = int(n_patches)

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib().fepll_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
