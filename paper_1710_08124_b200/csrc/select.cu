// Kernel (b) exact path + kernel (c): tree descent with FP64 scoring, and
// the Wiener estimates grouped by leaf.
//
// Scoring restates pkg/src/fepll/gmm.py:323-339 for the children of the
// patch's current node (pkg/src/fepll/tree.py:417-425):
//     c = z . U_child,  score = const + ||z||^2 / nu_tail + sum_j c_j^2 w_j
// with np.argmin's first-minimum tie-break over the stored child order.
// The children of a node are packed as one "group" (P x sum of ranks), so
// one warp computes every child's projection in a single pass over z.
#include "route.cuh"

namespace fepll {

constexpr int kSelWarps = 4;   // level kernel (smem: level table + per-warp rows)
constexpr int kWienerWarps = 8;
constexpr int kColsPerLane = kMaxGroupCols / 32;

// one warp: best child of node u for the patch in zs (smem); returns BFS id.
__device__ __forceinline__ int score_children_fp64(const PlanView& pv, int t, int u,
                                                   const double* zs, double sqv,
                                                   double* tv) {
  const int lane = lane_id();
  const int P = pv.P;
  const int width = pv.grp_width[u];
  const double* G = pv.grp_basis + pv.grp_off64[u];
  const double* w = pv.grp_sqw + (int64_t)t * pv.grp_cols_total + pv.grp_col_off[u];
  const int ncol = (width - lane + 31) >> 5;
  double acc[kColsPerLane];
#pragma unroll
  for (int k = 0; k < kColsPerLane; ++k) acc[k] = 0.0;
  for (int p = 0; p < P; ++p) {
    const double zp = zs[p];
    const double* row = G + (int64_t)p * width + lane;
#pragma unroll
    for (int k = 0; k < kColsPerLane; ++k)
      if (k < ncol) acc[k] = fma(zp, __ldg(row + 32 * k), acc[k]);
  }
#pragma unroll
  for (int k = 0; k < kColsPerLane; ++k)
    if (k < ncol) {
      const int j = lane + 32 * k;
      tv[j] = acc[k] * acc[k] * w[j];
    }
  __syncwarp();
  const int nk = pv.child_count[u];
  double best = INFINITY;
  int bestk = nk;
  if (lane < nk) {
    const int v = pv.child_list[pv.child_start[u] + lane];
    const int c0 = pv.child_col_off[v];
    const int r = pv.node_rank[v];
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += tv[c0 + j];
    const int64_t ti = (int64_t)t * pv.n_nodes + v;
    best = pv.node_const[ti] + sqv / pv.node_nu_tail[ti] + s;
    bestk = lane;
  }
  // first minimum in child order (np.argmin)
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
  return pv.child_list[pv.child_start[u] + bestk];
}

__global__ void route_init_kernel(int64_t n_total, int32_t* seg0, int32_t* cnt, int64_t* off,
                                  int64_t* leaf_base, int32_t* labels, int root_leaf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_total) {
    if (root_leaf >= 0) labels[i] = root_leaf; else seg0[i] = (int32_t)i;
  }
  if (i == 0) {
    cnt[0] = (int32_t)n_total;
    off[0] = 0;
    leaf_base[0] = 0;
  }
}

__global__ void __launch_bounds__(kSelWarps * 32)
select_level_fp64_kernel(PlanView pv, LevelArgs a, const double* __restrict__ Z64,
                         const double* __restrict__ sq) {
  __shared__ LevelSmem s;
  __shared__ double zbuf[kSelWarps][kMaxP];
  __shared__ double tbuf[kSelWarps][kMaxGroupCols];
  level_setup(pv, a, s);
  const int lane = lane_id();
  double* zs = zbuf[warp_id()];
  double* tv = tbuf[warp_id()];
  const int P = pv.P;
  for (int64_t item = (int64_t)blockIdx.x * kSelWarps + warp_id(); item < s.total;
       item += (int64_t)gridDim.x * kSelWarps) {
    int u, patch;
    level_item(a, s, item, u, patch);
    const double* zr = Z64 + (int64_t)patch * P;
    for (int p = lane; p < P; p += 32) zs[p] = zr[p];
    __syncwarp();
    const int v = score_children_fp64(pv, a.t, u, zs, sq[patch], tv);
    if (lane == 0) level_route(pv, a, s, v, patch);
    __syncwarp();
  }
}

// exact FP64 re-scoring of decisions the tensor-core epilogue could not
// certify (select_tc.cu): queue entries are (patch, node) pairs of level d.
__global__ void __launch_bounds__(kSelWarps * 32)
rescore_fp64_kernel(PlanView pv, LevelArgs a, const double* __restrict__ Z64,
                    const double* __restrict__ sq, const int32_t* __restrict__ queue,
                    const int32_t* __restrict__ queue_len) {
  __shared__ LevelSmem s;
  __shared__ double zbuf[kSelWarps][kMaxP];
  __shared__ double tbuf[kSelWarps][kMaxGroupCols];
  level_setup(pv, a, s);
  const int lane = lane_id();
  double* zs = zbuf[warp_id()];
  double* tv = tbuf[warp_id()];
  const int P = pv.P;
  const int total = queue_len[a.depth];
  for (int item = blockIdx.x * kSelWarps + warp_id(); item < total; item += gridDim.x * kSelWarps) {
    const int patch = queue[2 * item];
    const int u = queue[2 * item + 1];
    const double* zr = Z64 + (int64_t)patch * P;
    for (int p = lane; p < P; p += 32) zs[p] = zr[p];
    __syncwarp();
    const int v = score_children_fp64(pv, a.t, u, zs, sq[patch], tv);
    if (lane == 0) level_route(pv, a, s, v, patch);
    __syncwarp();
  }
}

int rescore_queue(Plan* p, const LevelArgs& a, const double* Z64, const double* sq,
                  const int32_t* queue, const int32_t* queue_len, cudaStream_t st) {
  rescore_fp64_kernel<<<2 * kSMs, kSelWarps * 32, 0, st>>>(p->v, a, Z64, sq, queue, queue_len);
  FEPLL_LAUNCH();
  return kOk;
}

// Wiener estimate per patch, iterating the leaf buckets so consecutive warps
// share the component basis (gmm.py:352-359: U((gamma-gamma_tail) c) + gamma_tail z).
__global__ void __launch_bounds__(kWienerWarps * 32)
wiener_fp64_kernel(PlanView pv, int t, const int32_t* __restrict__ leaf_nodes, int n_leaf_nodes,
                   const int32_t* __restrict__ cnt, const int64_t* __restrict__ off,
                   const int32_t* __restrict__ leafseg, const double* __restrict__ Z64,
                   double* __restrict__ Zhat) {
  __shared__ int64_t pre[kMaxLevelNodes + 1];
  __shared__ double zbuf[kWienerWarps][kMaxP];
  __shared__ double cbuf[kWienerWarps][kMaxP];
  for (int k = threadIdx.x; k < n_leaf_nodes; k += blockDim.x) pre[k + 1] = cnt[leaf_nodes[k]];
  __syncthreads();
  if (threadIdx.x == 0) {
    pre[0] = 0;
    for (int k = 0; k < n_leaf_nodes; ++k) pre[k + 1] += pre[k];
  }
  __syncthreads();
  const int64_t total = pre[n_leaf_nodes];
  const int lane = lane_id();
  const int P = pv.P;
  double* zs = zbuf[warp_id()];
  double* cs = cbuf[warp_id()];
  for (int64_t item = (int64_t)blockIdx.x * kWienerWarps + warp_id(); item < total;
       item += (int64_t)gridDim.x * kWienerWarps) {
    int lo = 0, hi = n_leaf_nodes;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= item) lo = mid; else hi = mid;
    }
    const int v = leaf_nodes[lo];
    const int patch = leafseg[off[v] + (item - pre[lo])];
    const int k = pv.leaf_index[v];
    const int r = pv.model_rank[k];
    const double* U = pv.model_basis + pv.model_off64[k];
    const double* shrink = pv.model_shrink + (int64_t)t * pv.model_cols_total + pv.model_col_off[k];
    const double gt = pv.model_gamma_tail[(int64_t)t * pv.K + k];
    const double* zr = Z64 + (int64_t)patch * P;
    for (int p = lane; p < P; p += 32) zs[p] = zr[p];
    __syncwarp();
    for (int j = lane; j < r; j += 32) {
      double c = 0.0;
      for (int p = 0; p < P; ++p) c = fma(zs[p], __ldg(U + (int64_t)p * r + j), c);
      cs[j] = c * shrink[j];
    }
    __syncwarp();
    double* out = Zhat + (int64_t)patch * P;
    for (int p = lane; p < P; p += 32) {
      const double* row = U + (int64_t)p * r;
      double e = 0.0;
      for (int j = 0; j < r; ++j) e = fma(cs[j], __ldg(row + j), e);
      out[p] = e + gt * zs[p];
    }
    __syncwarp();
  }
}

__global__ void leaf_counts_kernel(const int32_t* leaf_nodes, int n_leaf_nodes,
                                   const int32_t* leaf_index, const int32_t* cnt, int64_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_leaf_nodes) out[leaf_index[leaf_nodes[k]]] = cnt[leaf_nodes[k]];
}

// the tcgen05 level kernel lives in select_tc.cu
int select_level_tc(Plan* p, const LevelArgs& a, const float* Z32, const double* Z64,
                    const double* sq, double guard, cudaStream_t st);

LevelArgs make_level(Plan* p, int d, int t, int32_t* labels) {
  LevelArgs a;
  a.depth = d;
  a.lvl_begin = p->level_start[d];
  a.lvl_end = p->level_start[d + 1];
  a.nxt_begin = p->level_start[d + 1];
  a.nxt_end = p->level_start[d + 2];
  a.seg_in = p->rs.seg[d & 1];
  a.seg_out = p->rs.seg[(d + 1) & 1];
  a.leafseg = p->rs.leafseg;
  a.cnt = p->rs.cnt;
  a.off = p->rs.off;
  a.leaf_base = p->rs.leaf_base;
  a.labels = labels;
  a.t = t;
  return a;
}

}  // namespace fepll

using namespace fepll;

extern "C" int fepll_select(fepll_plan_t plan, int32_t t, const double* Z64, const float* Z32,
                            const double* sq, int64_t n_total, int32_t mode, double guard,
                            int32_t* labels, int64_t* leaf_counts, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && labels != nullptr && sq != nullptr, "select: bad arguments");
  FEPLL_REQUIRE(t >= 0 && t < p->v.T, "select: iteration index outside the beta schedule");
  FEPLL_REQUIRE(n_total >= 0 && n_total <= p->rs.cap, "select: patch count exceeds the reserved scratch");
  FEPLL_REQUIRE(mode == 0 || mode == 1, "select: unknown mode");
  FEPLL_REQUIRE(mode == 1 || Z64 != nullptr, "select: exact mode needs FP64 patches");
  FEPLL_REQUIRE(mode == 0 || (Z32 != nullptr && p->have_tc), "select: tensor mode needs FP32 patches and a tcgen05 plan");
  cudaStream_t st = (cudaStream_t)stream;
  p->last_n_total = (int)n_total;
  FEPLL_CUDA(cudaMemsetAsync(p->rs.cnt, 0, sizeof(int32_t) * p->v.n_nodes, st));
  FEPLL_CUDA(cudaMemsetAsync(p->rs.queue_len, 0, sizeof(int32_t) * kMaxDepth, st));
  if (n_total == 0) {
    if (leaf_counts) FEPLL_CUDA(cudaMemsetAsync(leaf_counts, 0, sizeof(int64_t) * p->v.K, st));
    return kOk;
  }
  const int root_leaf = p->child_count[0] == 0 ? 0 : -1;
  route_init_kernel<<<(unsigned)((n_total + 255) / 256), 256, 0, st>>>(
      n_total, p->rs.seg[0], p->rs.cnt, p->rs.off, p->rs.leaf_base, labels, root_leaf);
  FEPLL_LAUNCH();
  if (root_leaf >= 0) {
    // single-component model: every patch is at the only leaf
    leaf_counts_kernel<<<1, 32, 0, st>>>(p->d_leaf_nodes, p->n_leaf_nodes, p->v.leaf_index,
                                          p->rs.cnt, leaf_counts ? leaf_counts : (int64_t*)nullptr);
    FEPLL_LAUNCH();
    return kOk;
  }
  for (int d = 0; d < p->n_levels; ++d) {
    LevelArgs a = make_level(p, d, t, labels);
    if (mode == 1) {
      int rc = select_level_tc(p, a, Z32, Z64, sq, guard, st);
      if (rc) return rc;
    } else {
      select_level_fp64_kernel<<<grid_for(n_total, kSelWarps, 148 * 8), kSelWarps * 32, 0, st>>>(
          p->v, a, Z64, sq);
      FEPLL_LAUNCH();
    }
  }
  if (leaf_counts) {
    leaf_counts_kernel<<<(p->n_leaf_nodes + 127) / 128, 128, 0, st>>>(
        p->d_leaf_nodes, p->n_leaf_nodes, p->v.leaf_index, p->rs.cnt, leaf_counts);
    FEPLL_LAUNCH();
  }
  return kOk;
}

extern "C" int fepll_wiener(fepll_plan_t plan, int32_t t, const double* Z64, const int32_t* labels,
                            int64_t n_total, double* Zhat, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && Z64 != nullptr && Zhat != nullptr, "wiener: bad arguments");
  FEPLL_REQUIRE(t >= 0 && t < p->v.T, "wiener: iteration index outside the beta schedule");
  FEPLL_REQUIRE(n_total == p->last_n_total, "wiener: must follow fepll_select on the same patches");
  FEPLL_REQUIRE(p->n_leaf_nodes <= kMaxLevelNodes, "wiener: too many leaves");
  (void)labels;
  if (n_total == 0) return kOk;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->child_count[0] == 0) {
    // root is the only leaf: its bucket is the identity order
    FEPLL_CUDA(cudaMemsetAsync(p->rs.off, 0, sizeof(int64_t), st));
    route_init_kernel<<<(unsigned)((n_total + 255) / 256), 256, 0, st>>>(
        n_total, p->rs.leafseg, p->rs.cnt, p->rs.off, p->rs.leaf_base, (int32_t*)nullptr, -1);
    FEPLL_LAUNCH();
  }
  wiener_fp64_kernel<<<grid_for(n_total, kWienerWarps, 148 * 8), kWienerWarps * 32, 0, st>>>(
      p->v, t, p->d_leaf_nodes, p->n_leaf_nodes, p->rs.cnt, p->rs.off, p->rs.leafseg, Z64, Zhat);
  FEPLL_LAUNCH();
  return kOk;
}

extern "C" int fepll_select_rescored(fepll_plan_t plan, int32_t* dst, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && dst != nullptr, "select_rescored: bad arguments");
  FEPLL_CUDA(cudaMemcpyAsync(dst, p->rs.queue_len, sizeof(int32_t) * kMaxDepth,
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return kOk;
}
