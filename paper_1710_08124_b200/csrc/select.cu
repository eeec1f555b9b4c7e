// Kernel (b) exact path, the re-scoring kernel, and kernel (c) Wiener.
//
// Scoring restates pkg/src/fepll/gmm.py:323-339 for the children of the
// patch's current node (pkg/src/fepll/tree.py:417-425):
//     c = z . U_child,  score = const + ||z||^2 / nu_tail + sum_j c_j^2 w_j
// with np.argmin's first-minimum tie-break over the stored child order.
// The children of a node are packed as one "group" (P x sum of ranks), so
// one warp computes every child's projection in a single pass over z.
//
// Patches are never materialized in FP64: every kernel re-extracts z from the
// resident FP64 image as x[window] - dc — the exact operation of
// pkg/src/fepll/patches.py:178 — so the FP64 paths see the reference's
// patch values bit for bit.
#include <algorithm>

#include "fp64_score.cuh"

namespace fepll {

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
select_level_fp64_kernel(PlanView pv, LevelArgs a, PatchSrc ps, const double* __restrict__ sq) {
  __shared__ LevelTables s;
  __shared__ double zbuf[kSelWarps][kMaxP];
  __shared__ double tbuf[kSelWarps][kMaxGroupCols];
  level_tables(pv, a, s, 1);
  const int lane = lane_id();
  double* zs = zbuf[warp_id()];
  double* tv = tbuf[warp_id()];
  for (int item = blockIdx.x * kSelWarps + warp_id(); item < s.total_items;
       item += gridDim.x * kSelWarps) {
    int u, patch;
    level_item(a, s, item, u, patch);
    load_patch(ps, patch, pv.P, zs);
    const int v = score_children_fp64(pv, a.t, u, zs, sq[patch], tv);
    if (lane == 0) level_route(pv, a, s, v, patch);
    __syncwarp();
  }
}

// exact FP64 re-scoring of decisions the tensor-core epilogue could not
// certify: queue entries are (patch, node) pairs of level d.
// debug (fepll_debug_level_spans): earliest CTA entry / latest CTA exit
__device__ __forceinline__ void rs_span(uint64_t* sp, int slot) {
  if (sp && threadIdx.x == 0) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    if (slot == 0) atomicMin((unsigned long long*)sp, (unsigned long long)g);
    else atomicMax((unsigned long long*)sp + 1, (unsigned long long)g);
  }
}

__global__ void __launch_bounds__(kSelWarps * 32, 4)
rescore_fp64_kernel(PlanView pv, LevelArgs a, PatchSrc ps, const double* __restrict__ sq,
                    const int32_t* __restrict__ queue, const int32_t* __restrict__ queue_len,
                    uint64_t* sp) {
  pdl_wait();     // PDL behind the level kernel: its queue and counts
  pdl_trigger();  // the next level's prologue may overlap this grid
  rs_span(sp, 0);
  // The level kernel already published the next level's segment offsets in
  // a.off (route.cuh level_tables, CTA 0), so no per-CTA table rebuild here.
  __shared__ double zbuf[kSelWarps][kMaxP];
  __shared__ double tbuf[kSelWarps][kMaxGroupCols];
  const int lane = lane_id();
  double* zs = zbuf[warp_id()];
  double* tv = tbuf[warp_id()];
  const int total = queue_len[a.depth];
  for (int item = blockIdx.x * kSelWarps + warp_id(); item < total; item += gridDim.x * kSelWarps) {
    const int patch = queue[2 * item];
    const int u = queue[2 * item + 1];
    load_patch(ps, patch, pv.P, zs);
    const int v = score_children_fp64(pv, a.t, u, zs, sq[patch], tv);
    if (lane == 0) {
      const int slot = atomicAdd(&a.cnt[v], 1);
      if (pv.child_count[v] > 0) {
        a.seg_out[a.off[v] + slot] = patch;
        if (a.sq_out) a.sq_out[a.off[v] + slot] = sq[patch];
      } else {
        a.leafseg[a.off[v] + slot] = patch;
        a.labels[patch] = pv.leaf_index[v];
      }
    }
    __syncwarp();
  }
  __syncthreads();
  rs_span(sp, 1);
}

// Node-grouped form of rescore_fp64_kernel: CTA (k, j) takes the queued
// decisions of node u = lvl_begin + k (share j of gridDim.y), stages u's
// group matrix (P x width FP64, the children's bases side by side) in
// shared memory once, then scores each queued patch against it — the same
// FP64 operations in the same order as score_children_fp64 (bitwise the
// same scores), but one L2 read of the group per CTA instead of one per
// decision, and no dependent L2 round trips per row.  Used when the widest
// group of the level fits (kRescoreSmem).
constexpr int kRescoreWarps = 8;
constexpr int kRescoreChunk = 1024;  // queue entries compacted per pass
constexpr size_t kRescoreSmem = 160 * 1024;  // group matrix bytes (+ 48 KB of per-warp rows)
constexpr size_t kRescoreWarpSmem = sizeof(double) * kRescoreWarps * (kMaxP + kMaxGroupCols);

__global__ void __launch_bounds__(kRescoreWarps * 32, 1)
rescore_node_kernel(PlanView pv, LevelArgs a, PatchSrc ps, const double* __restrict__ sq,
                    const int32_t* __restrict__ queue, const int32_t* __restrict__ queue_len) {
  // dynamic: per-warp patch rows and score terms, then the [P][width] group
  // matrix of node u
  extern __shared__ __align__(16) double dyn[];
  double (*zbuf)[kMaxP] = reinterpret_cast<double (*)[kMaxP]>(dyn);
  double (*tbuf)[kMaxGroupCols] = reinterpret_cast<double (*)[kMaxGroupCols]>(dyn + kRescoreWarps * kMaxP);
  double* gs = dyn + kRescoreWarps * (kMaxP + kMaxGroupCols);
  __shared__ int32_t list[kRescoreChunk];
  __shared__ int32_t wcnt[kRescoreWarps];
  const int lane = lane_id(), warp = warp_id();
  const int total = queue_len[a.depth];
  const int u = a.lvl_begin + blockIdx.x;
  const int P = pv.P;
  const int width = pv.grp_width[u];
  const int nk = pv.child_count[u];
  if (total == 0 || nk == 0) return;
  const double* w = pv.grp_sqw + (int64_t)a.t * pv.grp_cols_total + pv.grp_col_off[u];
  const int32_t* kids = pv.child_list + pv.child_start[u];
  bool staged = false;
  int seen = 0;  // matches of node u in earlier chunks (share j takes match m with m % gridDim.y == j)
  for (int c0 = 0; c0 < total; c0 += kRescoreChunk) {
    const int c1 = min(total, c0 + kRescoreChunk);
    __syncthreads();  // the previous chunk's list is consumed
    // compaction of node u's entries in queue order: every thread tests
    // kPer entries (loads issued together), then per pass a warp ballot and
    // a prefix over the warps' counts
    constexpr int kPer = kRescoreChunk / (kRescoreWarps * 32);
    int2 ent[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = c0 + k * kRescoreWarps * 32 + threadIdx.x;
      ent[k] = i < c1 ? __ldg(reinterpret_cast<const int2*>(queue) + i) : make_int2(-1, -1);
    }
    int running = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const bool hit = ent[k].y == u;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) wcnt[warp] = __popc(m);
      __syncthreads();
      int before = running, pass = 0;
      for (int w2 = 0; w2 < kRescoreWarps; ++w2) {
        const int c = wcnt[w2];
        if (w2 < warp) before += c;
        pass += c;
      }
      if (hit) list[before + __popc(m & ((1u << lane) - 1u))] = ent[k].x;
      running += pass;
      __syncthreads();  // wcnt reused by the next pass
    }
    const int nl = running;
    // this share's items: global match index (seen + q) % gridDim.y == blockIdx.y
    const int first = (int)((blockIdx.y + gridDim.y - (unsigned)(seen % gridDim.y)) % gridDim.y);
    seen += nl;
    if (first >= nl) continue;
    if (!staged) {
      const int64_t nel = (int64_t)P * width;
      const double* G = pv.grp_basis + pv.grp_off64[u];
      for (int64_t e = threadIdx.x; e < nel; e += blockDim.x) gs[e] = __ldg(G + e);
      __syncthreads();
      staged = true;
    }
    double* zs = zbuf[warp];
    double* tv = tbuf[warp];
    for (int q = first + warp * gridDim.y; q < nl; q += kRescoreWarps * gridDim.y) {
      const int patch = list[q];
      load_patch(ps, patch, P, zs);
      if (width <= 128)
        child_terms<4, 8, true>(gs, w, width, width, P, zs, lane, tv);
      else if (width <= 256)
        child_terms<8, 4, true>(gs, w, width, width, P, zs, lane, tv);
      else
        child_terms<kColsPerLane, 2, true>(gs, w, width, width, P, zs, lane, tv);
      __syncwarp();
      double b;
      int bk;
      block_argmin(pv, a.t, u, 0, nk, 0, tv, sq[patch], b, bk);
      const int v = kids[bk];
      if (lane == 0) {
        const int slot = atomicAdd(&a.cnt[v], 1);
        if (pv.child_count[v] > 0) {
          a.seg_out[a.off[v] + slot] = patch;
          if (a.sq_out) a.sq_out[a.off[v] + slot] = sq[patch];
        } else {
          a.leafseg[a.off[v] + slot] = patch;
          a.labels[patch] = pv.leaf_index[v];
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// ---- deferred verification (plan option defer; ws2 trees).  The level
// kernels route an uncertified row by its tensor-core argmin like a
// certified one and log (patch, node, depth, provisional child); nothing
// waits between levels.  After the last level, verify_kernel re-scores every
// logged decision in FP64 (score_children_fp64: the arithmetic of the
// per-level re-scoring) and records the disagreements; the earliest one of a
// patch (first_bad) is where its path first left the FP64 argmin path — all
// its decisions before were certified or verified — so repair_kernel
// re-descends it from the FP64 child in FP64, leaves a hole (-1) in the
// provisional leaf bucket and appends it to the right one (leaf buckets hold
// a quarter of the parent's count + 32 spare slots, route.cuh
// leaf_capacity; an error flag past them).  Labels, leaf buckets and
// counts are those of re-scoring after every level.
__global__ void __launch_bounds__(kSelWarps * 32, 4)
verify_kernel(PlanView pv, int t, PatchSrc ps, const double* __restrict__ sq, const int4* __restrict__ vq,
              int32_t* vq_len, int64_t cap, int2* __restrict__ dq, int32_t* first_bad) {
  __shared__ double zbuf[kSelWarps][kMaxP];
  __shared__ double tbuf[kSelWarps][kMaxGroupCols];
  const int lane = lane_id();
  double* zs = zbuf[warp_id()];
  double* tv = tbuf[warp_id()];
  const int64_t total = min((int64_t)vq_len[0], cap);
  for (int64_t item = (int64_t)blockIdx.x * kSelWarps + warp_id(); item < total;
       item += (int64_t)gridDim.x * kSelWarps) {
    const int4 e = vq[item];
    load_patch(ps, e.x, pv.P, zs);
    const int v = score_children_fp64(pv, t, e.y, zs, sq[e.x], tv);
    if (lane == 0 && v != e.w) {
      atomicMin(&first_bad[e.x], e.z);
      const int slot = atomicAdd(&vq_len[1], 1);
      dq[slot] = make_int2(e.x, (e.z << 24) | v);
    }
    __syncwarp();
  }
}

// Repair with a CTA per mis-routed patch: the FP64 descent is a chain of
// one scoring per level, so each level's projection is split over the four
// warps (warp w: group columns w*32 + lane, + 128) — two 32-row chunks of
// G per level instead of eight 8-row ones — with the column chains, terms
// and first-minimum of score_children_fp64 / block_argmin (bitwise the same
// child).  Groups up to 256 columns and 32 children (every ws2 tree).
constexpr int kRpWarps = 4;

__global__ void __launch_bounds__(kRpWarps * 32)
repair_cta_kernel(PlanView pv, LevelArgs a, PatchSrc ps, const double* __restrict__ sq,
                  const int2* __restrict__ dq, const int32_t* __restrict__ vq_len, int32_t* first_bad,
                  const int32_t* __restrict__ pos_leaf, int32_t* holes, int32_t* flags) {
  __shared__ double zs[kMaxP];
  __shared__ double tv[256];
  __shared__ int s_v, s_go;
  const int lane = lane_id(), warp = warp_id();
  const int total = vq_len[1];
  const int P = pv.P;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int2 e = dq[item];
    const int g = e.x, d = e.y >> 24;
    // thread 0's read decides for the CTA (another CTA may reset first_bad[g])
    if (threadIdx.x == 0) s_go = first_bad[g] == d;
    __syncthreads();
    const bool go = s_go;
    __syncthreads();
    if (!go) continue;
    int v = e.y & 0xFFFFFF;
    if (warp == 0) load_patch(ps, g, P, zs);
    const double sqv = sq[g];
    __syncthreads();
    while (pv.child_count[v] > 0) {
      const int u = v;
      const int width = pv.grp_width[u];
      const int nk = pv.child_count[u];
      const double* G = pv.grp_basis + pv.grp_off64[u];
      const double* w = pv.grp_sqw + (int64_t)a.t * pv.grp_cols_total + pv.grp_col_off[u];
      double acc[2] = {0.0, 0.0};
      for (int p0 = 0; p0 < P; p0 += 32) {
        double gr[32][2];
#pragma unroll
        for (int r = 0; r < 32; ++r)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb) {
            const int col = cb * 128 + warp * 32 + lane;
            gr[r][cb] = (p0 + r < P && col < width) ? __ldg(G + (int64_t)(p0 + r) * width + col) : 0.0;
          }
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (p0 + r < P) {
            const double zp = zs[p0 + r];
            acc[0] = fma(zp, gr[r][0], acc[0]);
            acc[1] = fma(zp, gr[r][1], acc[1]);
          }
      }
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        const int col = cb * 128 + warp * 32 + lane;
        if (col < width) tv[col] = acc[cb] * acc[cb] * w[col];
      }
      __syncthreads();
      if (warp == 0) {
        double b;
        int bk;
        block_argmin(pv, a.t, u, 0, nk, 0, tv, sqv, b, bk);
        if (lane == 0) s_v = pv.child_list[pv.child_start[u] + bk];
      }
      __syncthreads();
      v = s_v;
    }
    if (threadIdx.x == 0) {
      a.leafseg[pos_leaf[g]] = -1;  // hole in the provisional bucket
      atomicAdd(&holes[a.labels[g]], 1);
      const int slot = atomicAdd(&a.cnt[v], 1);
      if (slot < leaf_capacity(a.cnt[pv.parent[v]])) {  // the bucket's capacity (route.cuh)
        a.leafseg[a.off[v] + slot] = g;
        a.labels[g] = pv.leaf_index[v];
      } else {
        atomicOr(flags, 2);
      }
      first_bad[g] = 0x7f7f7f7f;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSelWarps * 32, 4)
repair_kernel(PlanView pv, LevelArgs a, PatchSrc ps, const double* __restrict__ sq, const int2* __restrict__ dq,
              const int32_t* __restrict__ vq_len, int32_t* first_bad, const int32_t* __restrict__ pos_leaf,
              int32_t* holes, int32_t* flags) {
  __shared__ double zbuf[kSelWarps][kMaxP];
  __shared__ double tbuf[kSelWarps][kMaxGroupCols];
  const int lane = lane_id();
  double* zs = zbuf[warp_id()];
  double* tv = tbuf[warp_id()];
  const int total = vq_len[1];
  for (int item = blockIdx.x * kSelWarps + warp_id(); item < total; item += gridDim.x * kSelWarps) {
    const int2 e = dq[item];
    const int g = e.x, d = e.y >> 24;
    // a later entry of a patch already off the FP64 path; lane 0's read
    // decides for the warp (another warp may reset first_bad[g] meanwhile)
    if (__shfl_sync(0xffffffffu, first_bad[g], 0) != d) continue;
    int v = e.y & 0xFFFFFF;
    load_patch(ps, g, pv.P, zs);
    const double sqv = sq[g];
    while (pv.child_count[v] > 0) v = score_children_fp64(pv, a.t, v, zs, sqv, tv);
    if (lane == 0) {
      a.leafseg[pos_leaf[g]] = -1;  // hole in the provisional bucket
      atomicAdd(&holes[a.labels[g]], 1);
      const int slot = atomicAdd(&a.cnt[v], 1);
      if (slot < leaf_capacity(a.cnt[pv.parent[v]])) {  // the bucket's capacity (route.cuh)
        a.leafseg[a.off[v] + slot] = g;
        a.labels[g] = pv.leaf_index[v];
      } else {
        atomicOr(flags, 2);
      }
      first_bad[g] = 0x7f7f7f7f;
    }
    __syncwarp();
  }
}

// Wiener estimate per patch (fallback for large P / rank), iterating the leaf
// buckets (gmm.py:352-359: U((gamma-gamma_tail) c) + gamma_tail z).  Every
// Wiener kernel writes est + dc, the values patches.py:198-222 reprojects.
__global__ void __launch_bounds__(kWienerWarps * 32)
wiener_fp64_kernel(PlanView pv, int t, const int32_t* __restrict__ leaf_nodes, int n_leaf_nodes,
                   const int32_t* __restrict__ cnt, const int64_t* __restrict__ off,
                   const int32_t* __restrict__ leafseg, PatchSrc ps, double* __restrict__ Zhat) {
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
    load_patch(ps, patch, P, zs);
    for (int j = lane; j < r; j += 32) {
      double c = 0.0;
      for (int p = 0; p < P; ++p) c = fma(zs[p], __ldg(U + (int64_t)p * r + j), c);
      cs[j] = c * shrink[j];
    }
    __syncwarp();
    double* out = Zhat + ps.zrow(patch) * P;
    for (int p = lane; p < P; p += 32) {
      const double* row = U + (int64_t)p * r;
      double e = 0.0;
      for (int j = 0; j < r; ++j) e = fma(cs[j], __ldg(row + j), e);
      const double est = e + gt * zs[p];
      out[p] = ps.add_dc ? __dadd_rn(est, ps.dc[patch]) : est;  // reprojection input: est + dc
    }
    __syncwarp();
  }
}

// Tiled FP64 Wiener (gmm.py:352-359): a tile is up to 64 patches of one leaf
// component k (the leaf buckets of the last select).  The CTA stages Z
// (64 x P), U_k (P x r) and U_k^T in shared memory, then
//   C = (Z U_k) * shrink          (64 x r)
//   Zhat = C U_k^T + gamma_tail Z (64 x P)
// with 4x4 register blocks per thread.  FP64 throughout: the estimates feed
// the next iteration's tree decisions, which must stay those of the FP64
// reference.
constexpr int kWRows = 64;
constexpr int kWThreads = 256;

struct WienerSmemHead {
  int32_t tpre[kMaxLevelNodes + 1];
  uint64_t scan_tmp[256];
  int32_t rows[kWRows];
};

__global__ void __launch_bounds__(kWThreads)
wiener_tile_kernel(PlanView pv, int t, const int32_t* __restrict__ leaf_nodes, int n_leaf_nodes,
                   const int32_t* __restrict__ cnt, const int64_t* __restrict__ off,
                   const int32_t* __restrict__ leafseg, PatchSrc ps, double* __restrict__ Zhat,
                   int rmax) {
  extern __shared__ __align__(16) uint8_t wsm[];
  WienerSmemHead& h = *reinterpret_cast<WienerSmemHead*>(wsm);
  const int P = pv.P;
  const int zs_ld = P + 1;
  double* Zs = reinterpret_cast<double*>(wsm + ((sizeof(WienerSmemHead) + 15) & ~size_t(15)));
  double* Us = Zs + kWRows * zs_ld;        // [P][rmax]
  double* UT = Us + P * rmax;              // [rmax][P]
  double* Cs = UT + rmax * P;              // [64][rmax+1]
  double* sh = Cs + kWRows * (rmax + 1);   // [rmax]
  const int cs_ld = rmax + 1;
  const int tid = threadIdx.x;
  for (int k = tid; k < n_leaf_nodes; k += kWThreads)
    h.tpre[k] = (cnt[leaf_nodes[k]] + kWRows - 1) / kWRows;
  __syncthreads();
  const int tiles = block_exscan(h.tpre, n_leaf_nodes, h.scan_tmp);
  if (tid == 0) h.tpre[n_leaf_nodes] = tiles;
  __syncthreads();
  const int ig = tid >> 4;   // rows 4*ig .. 4*ig+3
  const int jg = tid & 15;   // columns jg + 16*c
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int li = prefix_find(h.tpre, n_leaf_nodes, tile);
    const int v = leaf_nodes[li];
    const int comp = pv.leaf_index[v];
    const int r = pv.model_rank[comp];
    const int first = (tile - h.tpre[li]) * kWRows;
    const int m = min(kWRows, cnt[v] - first);
    if (tid < kWRows) h.rows[tid] = tid < m ? leafseg[off[v] + first + tid] : -1;
    const double* U = pv.model_basis + pv.model_off64[comp];
    for (int e = tid; e < P * r; e += kWThreads) {
      const int p = e / r, j = e - p * r;
      const double u = U[e];
      Us[p * rmax + j] = u;
      UT[j * P + p] = u;
    }
    const double* shrink = pv.model_shrink + (int64_t)t * pv.model_cols_total + pv.model_col_off[comp];
    for (int j = tid; j < r; j += kWThreads) sh[j] = shrink[j];
    __syncthreads();
    for (int e = tid; e < kWRows * P; e += kWThreads) {
      const int i = e / P, p = e - i * P;
      const int g = h.rows[i];
      double z = 0.0;
      if (g >= 0) {
        const int b = g / ps.n_img;
        const int ia = g - b * ps.n_img;
        const int dr = p / ps.side;
        z = ps.x[((int64_t)b * ps.H + ps.anchors[2 * ia] + dr) * ps.W + ps.anchors[2 * ia + 1] +
                 (p - dr * ps.side)] - ps.dc[g];
      }
      Zs[i * zs_ld + p] = z;
    }
    __syncthreads();
    // C = (Z U) * shrink
    {
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      for (int p = 0; p < P; ++p) {
        double z[4], u[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) z[a] = Zs[(4 * ig + a) * zs_ld + p];
#pragma unroll
        for (int c = 0; c < 4; ++c) u[c] = (jg + 16 * c < r) ? Us[p * rmax + jg + 16 * c] : 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(z[a], u[c], acc[a][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = jg + 16 * c;
        if (j < r)
#pragma unroll
          for (int a = 0; a < 4; ++a) Cs[(4 * ig + a) * cs_ld + j] = acc[a][c] * sh[j];
      }
    }
    __syncthreads();
    // Zhat = C U^T + gamma_tail Z
    const double gt = pv.model_gamma_tail[(int64_t)t * pv.K + comp];
    for (int pc0 = 0; pc0 < P; pc0 += 64) {
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      for (int j = 0; j < r; ++j) {
        double cc[4], u[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) cc[a] = Cs[(4 * ig + a) * cs_ld + j];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int p = pc0 + jg + 16 * c;
          u[c] = p < P ? UT[j * P + p] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(cc[a], u[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = 4 * ig + a;
        const int row = h.rows[i];
        if (row < 0) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int p = pc0 + jg + 16 * c;
          if (p < P) {
            const double est = acc[a][c] + gt * Zs[i * zs_ld + p];
            Zhat[ps.zrow(row) * P + p] = ps.add_dc ? __dadd_rn(est, ps.dc[row]) : est;  // + dc
          }
        }
      }
    }
    __syncthreads();
  }
}

__global__ void leaf_counts_kernel(const int32_t* leaf_nodes, int n_leaf_nodes,
                                   const int32_t* leaf_index, const int32_t* cnt, const int32_t* holes,
                                   int64_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_leaf_nodes) {
    const int c = leaf_index[leaf_nodes[k]];
    out[c] = cnt[leaf_nodes[k]] - (holes ? holes[c] : 0);
  }
}

// tensor-core level kernels (select_tc.cu: K atoms streamed per tile, any
// P <= 128; select_ws.cu: warp-specialized pipeline, P <= 64)
int select_level_tc(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                    cudaStream_t st);
bool select_ws_supported(const Plan* p, int d);
int select_level_wide(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                      cudaStream_t st);
int select_level_ws2(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                     cudaStream_t st);
// Plan option select_variant: 0 select_ws.cu (3xTF32), 1 (default)
// select_ws2.cu (tf32 + bf16 cross pass, split loader / converter warps;
// measured faster on every level of the cfg5 tree), 2 ws2 on levels of
// <= 16 nodes, ws on the wider ones
int select_level_ws(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                    cudaStream_t st);

extern uint64_t* g_level_spans;

static int side_of(int P) {
  int s = 1;
  while (s * s < P) ++s;
  return s;
}

int rescore_queue_x(Plan* p, const LevelArgs& a, const double* x, const int32_t* anchors, int n_img,
                    int H, int W, const double* dc, const double* sq, const double* Z64,
                    cudaStream_t st) {
  PatchSrc ps{x, anchors, dc, n_img, H, W, side_of(p->v.P), n_img, Z64};
  const int nd = a.lvl_end - a.lvl_begin;
  uint64_t* sp = g_level_spans ? g_level_spans + (size_t)16 * kSMs * 4 + 2 * a.depth : nullptr;
  const size_t gbytes = sizeof(double) * (size_t)p->v.P * p->max_group_cols_at_depth[a.depth];
  if (p->opt.rescore_by_node && gbytes <= kRescoreSmem && !p->level_wide[a.depth]) {
    // node-grouped: the level's internal nodes x shares, ~two CTAs per SM
    const int shares = std::max(1, (2 * kSMs + nd - 1) / nd);
    FEPLL_CUDA(cudaFuncSetAttribute(rescore_node_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(kRescoreSmem + kRescoreWarpSmem)));
    rescore_node_kernel<<<dim3(nd, shares), kRescoreWarps * 32, kRescoreWarpSmem + gbytes, st>>>(
        p->v, a, ps, sq, p->rs.queue, p->rs.queue_len);
  } else {
    if (p->opt.pdl)
      FEPLL_CUDA(launch_pdl(rescore_fp64_kernel, dim3(4 * kSMs), dim3(kSelWarps * 32), 0, st, p->v, a, ps, sq,
                            (const int32_t*)p->rs.queue, (const int32_t*)p->rs.queue_len, sp));
    else
      rescore_fp64_kernel<<<4 * kSMs, kSelWarps * 32, 0, st>>>(p->v, a, ps, sq, p->rs.queue,
                                                               p->rs.queue_len, sp);
  }
  FEPLL_LAUNCH();
  return kOk;
}

int wiener_dmma(Plan* p, int t, const double* Z64, const double* dc, double* Zhat, int n_img,
                int zrows, const double* x, const int32_t* anchors, int H, int W, cudaStream_t st);
int wiener_dmma_f32(Plan* p, int t, const float* Z32, int z32_pitch, const double* dc, float* Zhat,
                    int n_img, int zrows, const double* x, const int32_t* anchors, int H, int W,
                    cudaStream_t st);
bool wiener_xw_supported(const Plan* p);
bool wiener_tc_supported(const Plan* p);
int wiener_tc_f32(Plan* p, int t, const float* Z32, int z32_pitch, const double* dc, float* Zhat, int n_img,
                  int zrows, cudaStream_t st);
bool wiener_dmma_supported(const Plan* p);

// every level runs the ws2 kernel (select_variant 1, no wide level): the
// deferred verification covers the whole tree
bool deferred_verify(const Plan* p) {
  // every level runs ws2 (select_variant 1, P <= 64) or select_tc (P <= 128,
  // the levels ws does not support) — both log their uncertified rows
  if (!p->opt.defer || p->opt.select_variant != 1 || p->v.P > 128) return false;
  for (int d = 0; d < p->n_levels; ++d) {
    if (p->level_wide[d] || p->level_tc_npad[d] > 256) return false;
    if (select_ws_supported(p, d) && p->v.tc_x == nullptr) return false;  // would run the 3xTF32 ws kernel
  }
  return true;
}

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

extern "C" int fepll_select(fepll_plan_t plan, int32_t t, const double* x, int32_t H, int32_t W,
                            const int32_t* anchors, int32_t n_img, const double* dc,
                            const double* sq, const float* Z32, const double* Z64,
                            int64_t n_total, int32_t mode,
                            double guard, int32_t* labels, int64_t* leaf_counts, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && labels != nullptr && sq != nullptr && x != nullptr &&
                    anchors != nullptr && dc != nullptr,
                "select: bad arguments");
  FEPLL_REQUIRE(t >= 0 && t < p->v.T, "select: iteration index outside the beta schedule");
  FEPLL_REQUIRE(n_total >= 0 && n_total <= p->rs.cap, "select: patch count exceeds the reserved scratch");
  FEPLL_REQUIRE(n_img >= 1 && n_total % n_img == 0, "select: n_total must be a multiple of n_img");
  FEPLL_REQUIRE(n_total * std::max({1, p->max_inner_children, p->max_leaf_children}) < (int64_t(1) << 32),
                "select: too many patches for 32-bit segment offsets");
  FEPLL_REQUIRE(mode == 0 || mode == 1, "select: unknown mode");
  FEPLL_REQUIRE(mode == 0 || (Z32 != nullptr && p->have_tc),
                "select: tensor mode needs a tcgen05 plan and the FP32 patch rows");
  cudaStream_t st = (cudaStream_t)stream;
  p->last_n_total = (int)n_total;
  FEPLL_CUDA(cudaMemsetAsync(p->rs.cnt, 0, sizeof(int32_t) * p->v.n_nodes, st));
  FEPLL_CUDA(cudaMemsetAsync(p->rs.queue_len, 0, sizeof(int32_t) * kMaxDepth, st));
  const bool defer = mode == 1 && deferred_verify(p);
  FEPLL_CUDA(cudaMemsetAsync(p->rs.vq_len, 0, sizeof(int32_t) * 2, st));
  if (defer) {
    FEPLL_CUDA(cudaMemsetAsync(p->rs.holes, 0, sizeof(int32_t) * p->v.K, st));
  }
  if (n_total == 0) {
    if (leaf_counts) FEPLL_CUDA(cudaMemsetAsync(leaf_counts, 0, sizeof(int64_t) * p->v.K, st));
    return kOk;
  }
  const int root_leaf = p->child_count[0] == 0 ? 0 : -1;
  route_init_kernel<<<(unsigned)((n_total + 255) / 256), 256, 0, st>>>(
      n_total, p->rs.seg[0], p->rs.cnt, p->rs.off, p->rs.leaf_base, labels, root_leaf);
  FEPLL_LAUNCH();
  if (root_leaf < 0) {
    PatchSrc ps{x, anchors, dc, n_img, H, W, side_of(p->v.P), n_img, Z64};
    // which levels run the ws2 kernel (the dispatch below): consecutive ws2
    // levels hand ||z||^2 over in segment order
    auto is_ws2 = [&](int d) {
      if (d < 0 || d >= p->n_levels || mode != 1 || p->v.P > 128) return false;
      const bool wide = p->level_wide[d] || p->level_tc_npad[d] > 256;
      return !wide && select_ws_supported(p, d) && p->v.tc_x != nullptr &&
             (p->opt.select_variant == 1 ||
              (p->opt.select_variant == 2 && p->level_start[d + 1] - p->level_start[d] <= 16));
    };
    for (int d = 0; d < p->n_levels; ++d) {
      LevelArgs a = make_level(p, d, t, labels);
      if (p->opt.seg_sq && is_ws2(d)) {
        a.sq_in = d == 0 ? sq : is_ws2(d - 1) ? p->rs.segsq[d & 1] : nullptr;
        a.sq_out = is_ws2(d + 1) ? p->rs.segsq[(d + 1) & 1] : nullptr;
      }
      int rc = kOk;
      const bool prof = p->prof_used < (int)p->prof_ev.size() / 2;
      if (prof) FEPLL_CUDA(cudaEventRecord(p->prof_ev[2 * p->prof_used], st));
      if (mode == 1 && p->v.P <= 128) {
        // wide levels (the exhaustive star root) stream their columns in chunks
        const bool wide = p->level_wide[d] || p->level_tc_npad[d] > 256;
        rc = wide ? select_level_wide(p, a, Z32, sq, guard, st)
             : select_ws_supported(p, d)
                 ? ((p->v.tc_x != nullptr &&
                     (p->opt.select_variant == 1 ||
                      (p->opt.select_variant == 2 && p->level_start[d + 1] - p->level_start[d] <= 16)))
                        ? select_level_ws2(p, a, Z32, sq, guard, st)
                        : select_level_ws(p, a, Z32, sq, guard, st))
                 : select_level_tc(p, a, Z32, sq, guard, st);
        if (prof) FEPLL_CUDA(cudaEventRecord(p->prof_ev[2 * p->prof_used++ + 1], st));
        if (!rc && !defer) rc = rescore_queue_x(p, a, x, anchors, n_img, H, W, dc, sq, Z64, st);
      } else {  // exact mode, or P > 128 (beyond the tcgen05 kernels' K atoms):
                // FP64 scoring (wide nodes: block-wise scan) — the same labels
        select_level_fp64_kernel<<<grid_for(n_total, kSelWarps, 148 * 8), kSelWarps * 32, 0, st>>>(
            p->v, a, ps, sq);
        FEPLL_LAUNCH();
        if (prof) FEPLL_CUDA(cudaEventRecord(p->prof_ev[2 * p->prof_used++ + 1], st));
      }
      if (rc) return rc;
    }
    if (defer) {
      LevelArgs a = make_level(p, 0, t, labels);
      verify_kernel<<<4 * kSMs, kSelWarps * 32, 0, st>>>(p->v, t, ps, sq, p->rs.vq, p->rs.vq_len, p->rs.vq_cap,
                                                         p->rs.dq, p->rs.first_bad);
      FEPLL_LAUNCH();
      if (p->max_group_cols <= 256 && p->max_inner_children <= 32 && p->max_leaf_children <= 32)
        repair_cta_kernel<<<2 * kSMs, kRpWarps * 32, 0, st>>>(p->v, a, ps, sq, p->rs.dq, p->rs.vq_len,
                                                             p->rs.first_bad, p->rs.pos_leaf, p->rs.holes,
                                                             &p->rs.queue_len[kMaxDepth - 1]);
      else
        repair_kernel<<<kSMs, kSelWarps * 32, 0, st>>>(p->v, a, ps, sq, p->rs.dq, p->rs.vq_len, p->rs.first_bad,
                                                       p->rs.pos_leaf, p->rs.holes, &p->rs.queue_len[kMaxDepth - 1]);
      FEPLL_LAUNCH();
    }
  }
  if (leaf_counts) {
    leaf_counts_kernel<<<(p->n_leaf_nodes + 127) / 128, 128, 0, st>>>(
        p->d_leaf_nodes, p->n_leaf_nodes, p->v.leaf_index, p->rs.cnt, defer ? p->rs.holes : nullptr,
        leaf_counts);
    FEPLL_LAUNCH();
  }
  return kOk;
}

extern "C" int fepll_wiener_reads_image(fepll_plan_t plan) {
  return fepll::wiener_xw_supported(reinterpret_cast<fepll::Plan*>(plan)) ? 1 : 0;
}

extern "C" int fepll_select_rescored(fepll_plan_t plan, int32_t* dst, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && dst != nullptr, "select_rescored: bad arguments");
  FEPLL_CUDA(cudaMemcpyAsync(dst, p->rs.queue_len, sizeof(int32_t) * (kMaxDepth - 2),
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  // [62]: patches the deferred verification re-descended; [63]: its flags
  FEPLL_CUDA(cudaMemcpyAsync(dst + kMaxDepth - 2, p->rs.vq_len + 1, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
  FEPLL_CUDA(cudaMemcpyAsync(dst + kMaxDepth - 1, p->rs.queue_len + kMaxDepth - 1, sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return kOk;
}

extern "C" int fepll_wiener(fepll_plan_t plan, int32_t t, const double* x, int32_t H, int32_t W,
                            const int32_t* anchors, int32_t n_img, const double* dc,
                            const double* Z64, int64_t n_total, double* Zhat, int32_t zhat_rows,
                            void* stream) {
  using namespace fepll;
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && x != nullptr && anchors != nullptr && dc != nullptr &&
                    Zhat != nullptr,
                "wiener: bad arguments");
  FEPLL_REQUIRE(t >= 0 && t < p->v.T, "wiener: iteration index outside the beta schedule");
  FEPLL_REQUIRE(n_total == p->last_n_total, "wiener: must follow fepll_select on the same patches");
  FEPLL_REQUIRE(n_img >= 1 && zhat_rows >= n_img, "wiener: Zhat rows per image below n_img");
  FEPLL_REQUIRE(p->n_leaf_nodes <= kMaxLevelNodes, "wiener: too many leaves");
  if (n_total == 0) return kOk;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->child_count[0] == 0) {
    // root is the only leaf: its bucket is the identity order
    route_init_kernel<<<(unsigned)((n_total + 255) / 256), 256, 0, st>>>(
        n_total, p->rs.leafseg, p->rs.cnt, p->rs.off, p->rs.leaf_base, (int32_t*)nullptr, -1);
    FEPLL_LAUNCH();
  }
  if (wiener_dmma_supported(p) && (Z64 != nullptr || wiener_xw_supported(p)))
    return wiener_dmma(p, t, Z64, dc, Zhat, n_img, zhat_rows, x, anchors, H, W, st);
  PatchSrc ps{x, anchors, dc, n_img, H, W, side_of(p->v.P), zhat_rows};
  ps.add_dc = p->opt.wiener_add_dc;
  const int P = p->v.P;
  const int rmax = p->max_model_rank;
  if (rmax <= 64) {
    const size_t smem = ((sizeof(WienerSmemHead) + 15) & ~size_t(15)) +
                        sizeof(double) * ((size_t)kWRows * (P + 1) + 2 * (size_t)P * rmax +
                                          (size_t)kWRows * (rmax + 1) + rmax);
    FEPLL_CUDA(cudaFuncSetAttribute(wiener_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    wiener_tile_kernel<<<kSMs * 2, kWThreads, smem, st>>>(p->v, t, p->d_leaf_nodes, p->n_leaf_nodes,
                                                          p->rs.cnt, p->rs.off, p->rs.leafseg, ps,
                                                          Zhat, rmax);
  } else {
    wiener_fp64_kernel<<<grid_for(n_total, kWienerWarps, 148 * 8), kWienerWarps * 32, 0, st>>>(
        p->v, t, p->d_leaf_nodes, p->n_leaf_nodes, p->rs.cnt, p->rs.off, p->rs.leafseg, ps, Zhat);
  }
  FEPLL_LAUNCH();
  return kOk;
}

// FP32-state form of fepll_wiener: the FP32 patch rows of fepll_extract in
// (z32_pitch floats per row), est + dc rounded once to FP32 out; FP64
// arithmetic in between (DMMA).
extern "C" int fepll_wiener_f32(fepll_plan_t plan, int32_t t, const double* x, int32_t H, int32_t W,
                                const int32_t* anchors, int32_t n_img, const double* dc,
                                const float* Z32, int32_t z32_pitch, int64_t n_total, float* Zhat,
                                int32_t zhat_rows, void* stream) {
  using namespace fepll;
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && dc != nullptr && Z32 != nullptr && Zhat != nullptr,
                "wiener_f32: bad arguments");
  FEPLL_REQUIRE(t >= 0 && t < p->v.T, "wiener_f32: iteration index outside the beta schedule");
  FEPLL_REQUIRE(n_total == p->last_n_total, "wiener_f32: must follow fepll_select on the same patches");
  FEPLL_REQUIRE(n_img >= 1 && zhat_rows >= n_img, "wiener_f32: Zhat rows per image below n_img");
  FEPLL_REQUIRE(wiener_dmma_supported(p), "wiener_f32: patch size / rank outside the DMMA kernel");
  FEPLL_REQUIRE(z32_pitch >= p->v.P && z32_pitch % 4 == 0 && p->v.P % 4 == 0 &&
                    reinterpret_cast<uintptr_t>(Z32) % 16 == 0,
                "wiener_f32: FP32 rows need a pitch >= P, a multiple of 4, and 16-byte alignment");
  FEPLL_REQUIRE(p->opt.wiener_add_dc, "wiener_f32: writes est + dc only");
  if (n_total == 0) return kOk;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->child_count[0] == 0) {
    route_init_kernel<<<(unsigned)((n_total + 255) / 256), 256, 0, st>>>(
        n_total, p->rs.leafseg, p->rs.cnt, p->rs.off, p->rs.leaf_base, (int32_t*)nullptr, -1);
    FEPLL_LAUNCH();
  }
  if (p->opt.wiener_tc && wiener_tc_supported(p) && z32_pitch == (p->v.P + 31) / 32 * 32)
    return wiener_tc_f32(p, t, Z32, z32_pitch, dc, Zhat, n_img, zhat_rows, st);
  return wiener_dmma_f32(p, t, Z32, z32_pitch, dc, Zhat, n_img, zhat_rows, x, anchors, H, W, st);
}
