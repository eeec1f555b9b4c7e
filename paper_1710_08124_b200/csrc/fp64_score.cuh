// FP64 scoring of a patch against the children of its current node — the
// exact path of kernel (b) (select.cu: exact levels and re-scoring; the ws2
// tree-level kernel's in-kernel re-scoring tail).
//
// Restates pkg/src/fepll/gmm.py:323-339 for the children of the patch's
// current node (pkg/src/fepll/tree.py:417-425):
//     c = z . U_child,  score = const + ||z||^2 / nu_tail + sum_j c_j^2 w_j
// with np.argmin's first-minimum tie-break over the stored child order.
// The children of a node are packed as one "group" (P x sum of ranks), so
// one warp computes every child's projection in a single pass over z.
#pragma once
#include "route.cuh"

namespace fepll {

constexpr int kSelWarps = 4;   // level/rescore kernels (smem: level table + per-warp rows)
constexpr int kWienerWarps = 8;
constexpr int kColsPerLane = kMaxGroupCols / 32;

struct PatchSrc {
  const double* x;        // [B][H][W]
  const int32_t* anchors; // [n_img][2]
  const double* dc;       // [B*n_img]
  int n_img, H, W, side;
  int zrows;              // Zhat rows per image (>= n_img; padded pitch)
  const double* z64 = nullptr;  // FP64 patch rows of fepll_extract (bitwise window - dc), or NULL
  int add_dc = 1;               // Wiener output: est + dc (1) or the bare estimates (0)
  __device__ __forceinline__ int64_t zrow(int g) const {
    return zrows == n_img ? (int64_t)g : (int64_t)(g / n_img) * zrows + g % n_img;
  }
};

// warp: zs[0..P) = window(g) - dc[g]
__device__ __forceinline__ void load_patch(const PatchSrc& ps, int g, int P, double* zs) {
  if (ps.z64) {  // the extracted row: one round trip instead of anchors -> image -> dc
    for (int p = lane_id(); p < P; p += 32) zs[p] = ps.z64[(int64_t)g * P + p];
    __syncwarp();
    return;
  }
  const int b = g / ps.n_img;
  const int ia = g - b * ps.n_img;
  const int pr = ps.anchors[2 * ia], pc = ps.anchors[2 * ia + 1];
  const double* src = ps.x + ((int64_t)b * ps.H + pr) * ps.W + pc;
  const double d = ps.dc[g];
  for (int p = lane_id(); p < P; p += 32) {
    const int dr = p / ps.side;
    zs[p] = src[(int64_t)dr * ps.W + (p - dr * ps.side)] - d;
  }
  __syncwarp();
}

// lane's columns (lane + 32k, k < NC) of z . G for a P x ncols block of a
// row-major matrix with row stride `stride`, p ascending per column (one FMA
// chain each, the same order for every width); CH rows of G are loaded
// before they are consumed so a warp keeps CH*NC loads in flight instead of
// one L2 round trip per row.
template <int NC, int CH, bool kShared = false>
__device__ __forceinline__ void project_cols(const double* G, int stride, int ncols, int P,
                                             const double* zs, int lane, double (&acc)[NC]) {
  const int ncol = (ncols - lane + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = 0.0;
  int p = 0;
  for (; p + CH <= P; p += CH) {
    double g[CH][NC];
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int k = 0; k < NC; ++k)
        g[j][k] = k < ncol ? (kShared ? G[(int64_t)(p + j) * stride + lane + 32 * k]
                                      : __ldg(G + (int64_t)(p + j) * stride + lane + 32 * k))
                           : 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const double zp = zs[p + j];
#pragma unroll
      for (int k = 0; k < NC; ++k) acc[k] = fma(zp, g[j][k], acc[k]);
    }
  }
  for (; p < P; ++p) {
    const double zp = zs[p];
#pragma unroll
    for (int k = 0; k < NC; ++k)
      if (k < ncol)
        acc[k] = fma(zp, kShared ? G[(int64_t)p * stride + lane + 32 * k]
                                 : __ldg(G + (int64_t)p * stride + lane + 32 * k), acc[k]);
  }
}

// tv[j] = c_j^2 w_j for the ncols columns of the block (c = z . G)
template <int NC, int CH, bool kShared = false>
__device__ __forceinline__ void child_terms(const double* G, const double* w, int stride, int ncols,
                                            int P, const double* zs, int lane, double* tv) {
  double acc[NC];
  project_cols<NC, CH, kShared>(G, stride, ncols, P, zs, lane, acc);
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int j = lane + 32 * k;
    if (j < ncols) tv[j] = acc[k] * acc[k] * w[j];
  }
}

__device__ __forceinline__ void block_terms(const double* G, const double* w, int stride, int ncols,
                                            int P, const double* zs, int lane, double* tv) {
  if (ncols <= 128)
    child_terms<4, 8>(G, w, stride, ncols, P, zs, lane, tv);
  else if (ncols <= 256)
    child_terms<8, 4>(G, w, stride, ncols, P, zs, lane, tv);
  else
    child_terms<kColsPerLane, 2>(G, w, stride, ncols, P, zs, lane, tv);
  __syncwarp();
}

// children [k0, k1) of node u (k1 - k0 <= 32, columns [col0, col0 + tv
// width) already in tv): lane k - k0 scores child k; first minimum in child
// order (np.argmin) over the block
__device__ __forceinline__ void block_argmin(const PlanView& pv, int t, int u, int k0, int k1,
                                             int col0, const double* tv, double sqv,
                                             double& best, int& bestk) {
  const int lane = lane_id();
  best = INFINITY;
  bestk = k1;
  if (lane < k1 - k0) {
    const int v = pv.child_list[pv.child_start[u] + k0 + lane];
    const int c0 = pv.child_col_off[v] - col0;
    const int r = pv.node_rank[v];
    double sacc = 0.0;
    for (int j = 0; j < r; ++j) sacc += tv[c0 + j];
    const int64_t ti = (int64_t)t * pv.n_nodes + v;
    best = pv.node_const[ti] + sqv / pv.node_nu_tail[ti] + sacc;
    if (best != best) best = INFINITY;  // non-finite patch: still a valid child (status flags it)
    bestk = k0 + lane;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int ok = __shfl_xor_sync(0xffffffffu, bestk, o);
    if (ob < best || (ob == best && ok < bestk)) {
      best = ob;
      bestk = ok;
    }
  }
  __syncwarp();
}

// one warp: best child of node u for the patch in zs (smem); returns BFS id.
// A node within the single-pass limits (<= 32 children, <= 512 group
// columns) is one block; a wider one (the exhaustive star root of
// gmm.py:371-391, K children) is scanned in consecutive blocks with a
// strict-less running minimum, so ties still go to the lowest child index.
__device__ __forceinline__ int score_children_fp64(const PlanView& pv, int t, int u,
                                                   const double* zs, double sqv, double* tv) {
  const int lane = lane_id();
  const int P = pv.P;
  const int width = pv.grp_width[u];
  const int nk = pv.child_count[u];
  const double* G = pv.grp_basis + pv.grp_off64[u];
  const double* w = pv.grp_sqw + (int64_t)t * pv.grp_cols_total + pv.grp_col_off[u];
  const int32_t* kids = pv.child_list + pv.child_start[u];
  double best = INFINITY;
  int bestk = 0;
  // one block of all children when they fit (width = sum of the child ranks,
  // plan.py): the block split below walks the children with two dependent
  // loads each, the longest chain of the re-scoring kernel
  const bool one_block = nk <= 32 && width <= kMaxGroupCols;
  for (int k0 = 0; k0 < nk;) {
    int col0 = 0, k1 = nk, cols = width;
    if (!one_block) {
      col0 = pv.child_col_off[kids[k0]];
      k1 = k0;
      cols = 0;
      while (k1 < nk && k1 - k0 < 32 && cols + pv.node_rank[kids[k1]] <= kMaxGroupCols)
        cols += pv.node_rank[kids[k1++]];
    }
    block_terms(G + col0, w + col0, width, cols, P, zs, lane, tv);
    double b;
    int bk;
    block_argmin(pv, t, u, k0, k1, col0, tv, sqv, b, bk);
    if (b < best || k0 == 0) {
      best = b;
      bestk = bk;
    }
    k0 = k1;
  }
  return kids[bestk];
}


// score_children_fp64 for a node whose group fits one 128-column block (nk
// <= 32, width <= 128: the ws2 kernel's nodes) — the same operations in the
// same order (child_terms<4, 8>), with the registers of that case only
__device__ __forceinline__ int score_children_fp64_w128(const PlanView& pv, int t, int u,
                                                        const double* zs, double sqv, double* tv) {
  const int lane = lane_id();
  const int width = pv.grp_width[u];
  const int nk = pv.child_count[u];
  const double* G = pv.grp_basis + pv.grp_off64[u];
  const double* w = pv.grp_sqw + (int64_t)t * pv.grp_cols_total + pv.grp_col_off[u];
  child_terms<4, 8>(G, w, width, width, pv.P, zs, lane, tv);
  __syncwarp();
  double b;
  int bk;
  block_argmin(pv, t, u, 0, nk, 0, tv, sqv, b, bk);
  return pv.child_list[pv.child_start[u] + bk];
}

// route patch g to child v of the next level (segment / leaf bucket),
// one lane; the level kernel published a.off for the depth-(d+1) nodes
__device__ __forceinline__ void route_fp64_decision(const PlanView& pv, const LevelArgs& a, int v, int g,
                                                    double sqv) {
  const int slot = atomicAdd(&a.cnt[v], 1);
  if (pv.child_count[v] > 0) {
    a.seg_out[a.off[v] + slot] = g;
    if (a.sq_out) a.sq_out[a.off[v] + slot] = sqv;
  } else {
    a.leafseg[a.off[v] + slot] = g;
    a.labels[g] = pv.leaf_index[v];
  }
}

}  // namespace fepll
