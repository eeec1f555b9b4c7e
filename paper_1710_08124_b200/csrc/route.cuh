// Level-synchronous routing for the tree walk.
//
// The reference descends with a Python loop over the distinct nodes of each
// level (pkg/src/fepll/tree.py:416-428).  Here every level is one pass over
// the patches grouped by their current node ("segments"): a patch that picks
// child v is appended (atomic slot) to v's segment of the next level.
// Segment capacity of a child = its parent's count, so the next level's
// offsets are a prefix sum over the (at most a few hundred) nodes of the
// level, recomputed by every CTA from the final counts with a block scan —
// no global scan pass.  Leaves get buckets in a separate buffer; their
// counts are the label histogram used for Wiener grouping and the counters.
#pragma once
#include "plan.cuh"

namespace fepll {

constexpr int kMaxLevelNodes = 512;  // nodes per depth handled in smem

struct LevelArgs {
  int depth;
  int lvl_begin, lvl_end;   // BFS ids of depth-d nodes
  int nxt_begin, nxt_end;   // BFS ids of depth-(d+1) nodes
  const int32_t* seg_in;
  int32_t* seg_out;
  int32_t* leafseg;
  int32_t* cnt;
  int64_t* off;
  int64_t* leaf_base;
  int32_t* labels;
  int t;
  // ||z||^2 in segment order (ws2 levels): read at the rows' segment
  // positions instead of a random 8-byte gather sq[patch], written next to
  // the routed index for the next level; nullptr = not kept
  const double* sq_in = nullptr;
  double* sq_out = nullptr;
};

template <int NMAX>
struct LevelTablesN {
  static constexpr int kCap = NMAX;
  int32_t cpre[NMAX + 1];   // prefix of counts over depth-d internal nodes
  int32_t tpre[NMAX + 1];   // prefix of tiles (rows_per_tile) over the same
  int64_t child_off[NMAX];  // next-level segment offsets of depth-(d+1) nodes
  uint64_t scan_tmp[256];
  int32_t total_items;
  int32_t total_tiles;
};
using LevelTables = LevelTablesN<kMaxLevelNodes>;

// in-place exclusive scan of data[0..n) (smem) by the first <=255 threads;
// every thread of the block must call it.  Returns the total.  The <=255
// per-thread partial sums are scanned by warp 0 with shuffles (8 per lane):
// a serial scan by one thread cost ~4 us per call — three per tree-level
// launch, in every CTA, before its first row load.
template <typename T>
__device__ __forceinline__ T block_exscan(T* data, int n, uint64_t* tmp) {
  const int nt = min((int)blockDim.x, 255);
  const bool act = (int)threadIdx.x < nt;
  const int per = (n + nt - 1) / nt;
  const int b = threadIdx.x * per, e = act ? min(n, b + per) : b;
  T s = 0;
  for (int i = b; i < e; ++i) s += data[i];
  if (act) tmp[threadIdx.x] = (uint64_t)s;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint64_t v[8];
    uint64_t sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane * 8 + j;
      v[j] = i < nt ? tmp[i] : 0;
      sum += v[j];
    }
    uint64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    uint64_t run = incl - sum;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane * 8 + j;
      if (i < nt) tmp[i] = run;
      run += v[j];
    }
    if (lane == 31) tmp[nt] = incl;
  }
  __syncthreads();
  if (act) {
    T pre = (T)tmp[threadIdx.x];
    for (int i = b; i < e; ++i) {
      const T v = data[i];
      data[i] = pre;
      pre += v;
    }
  }
  const T total = (T)tmp[nt];
  __syncthreads();
  return total;
}

// Every CTA: count/tile prefixes of level d and the offsets of level d+1.
// capacity of a leaf bucket whose parent holds c patches: c plus spare
// slots for patches the deferred verification re-routes into it
__host__ __device__ __forceinline__ int leaf_capacity(int c) { return c + c / 4 + kLeafSlack; }

template <class LT>
__device__ inline void level_tables(const PlanView& pv, const LevelArgs& a, LT& s,
                                    int rows_per_tile) {
  const int nd = a.lvl_end - a.lvl_begin;
  const int nn = a.nxt_end - a.nxt_begin;
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const int u = a.lvl_begin + k;
    const int c = pv.child_count[u] > 0 ? a.cnt[u] : 0;
    s.cpre[k] = c;
    s.tpre[k] = (c + rows_per_tile - 1) / rows_per_tile;
  }
  // packed (leaf capacity << 32 | internal capacity) per next-level node
  uint64_t* cap = reinterpret_cast<uint64_t*>(s.child_off);
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const int v = a.nxt_begin + k;
    const uint64_t c = (uint64_t)(uint32_t)a.cnt[pv.parent[v]];
    cap[k] = pv.child_count[v] > 0 ? c : ((uint64_t)leaf_capacity((int)c) << 32);
  }
  __syncthreads();
  const int32_t items = block_exscan(s.cpre, nd, s.scan_tmp);
  const int32_t tiles = block_exscan(s.tpre, nd, s.scan_tmp);
  const uint64_t tot = block_exscan(cap, nn, s.scan_tmp);
  const int64_t lb = a.leaf_base[a.depth];
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const int v = a.nxt_begin + k;
    const uint64_t pre = cap[k];
    s.child_off[k] = pv.child_count[v] > 0 ? (int64_t)(pre & 0xffffffffull)
                                           : lb + (int64_t)(pre >> 32);
  }
  if (threadIdx.x == 0) {
    s.cpre[nd] = items;
    s.tpre[nd] = tiles;
    s.total_items = items;
    s.total_tiles = tiles;
    if (blockIdx.x == 0) a.leaf_base[a.depth + 1] = lb + (int64_t)(tot >> 32);
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < nn; k += blockDim.x) a.off[a.nxt_begin + k] = s.child_off[k];
}

// level_tables for levels of at most 256 nodes on both sides (every level the
// ws2 kernel takes): warp 0 computes the three prefix sums with eight entries
// per lane and shuffle scans, so the CTA meets one barrier instead of a
// dozen — the same tables bit for bit.  On small images the tree walk is
// launch- and prologue-bound (a 256^2 image has 33 tiles per level), and the
// prologue was mostly these barriers.  Every thread calls it; ends with a
// __syncthreads.
template <class LT>
__device__ inline void level_tables_warp(const PlanView& pv, const LevelArgs& a, LT& s,
                                         int rows_per_tile) {
  const int nd = a.lvl_end - a.lvl_begin;
  const int nn = a.nxt_end - a.nxt_begin;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    // counts and tiles of the depth-d internal nodes
    int c[8], tl[8];
    int sc = 0, st = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = 8 * lane + q;
      c[q] = 0;
      if (k < nd) {
        const int u = a.lvl_begin + k;
        c[q] = pv.child_count[u] > 0 ? a.cnt[u] : 0;
      }
      tl[q] = (c[q] + rows_per_tile - 1) / rows_per_tile;
      sc += c[q];
      st += tl[q];
    }
    // capacities of the depth-(d+1) nodes: (leaf << 32 | internal)
    uint64_t cap[8];
    uint64_t scap = 0;
    bool leaf[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = 8 * lane + q;
      cap[q] = 0;
      leaf[q] = false;
      if (k < nn) {
        const int v = a.nxt_begin + k;
        const uint64_t pc = (uint64_t)(uint32_t)a.cnt[pv.parent[v]];
        leaf[q] = pv.child_count[v] == 0;
        cap[q] = leaf[q] ? ((uint64_t)leaf_capacity((int)pc) << 32) : pc;
      }
      scap += cap[q];
    }
    const int64_t lb = a.leaf_base[a.depth];
    int ic = sc, it = st;
    uint64_t icap = scap;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yc = __shfl_up_sync(0xffffffffu, ic, o);
      const int yt = __shfl_up_sync(0xffffffffu, it, o);
      const uint64_t yp = __shfl_up_sync(0xffffffffu, icap, o);
      if (lane >= o) {
        ic += yc;
        it += yt;
        icap += yp;
      }
    }
    const int items = __shfl_sync(0xffffffffu, ic, 31), tiles = __shfl_sync(0xffffffffu, it, 31);
    const uint64_t tot = __shfl_sync(0xffffffffu, icap, 31);
    int rc = ic - sc, rt = it - st;
    uint64_t rp = icap - scap;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = 8 * lane + q;
      if (k < nd) {
        s.cpre[k] = rc;
        s.tpre[k] = rt;
      }
      rc += c[q];
      rt += tl[q];
      if (k < nn) {
        const int64_t o = leaf[q] ? lb + (int64_t)(rp >> 32) : (int64_t)(rp & 0xffffffffull);
        s.child_off[k] = o;
        if (blockIdx.x == 0) a.off[a.nxt_begin + k] = o;
      }
      rp += cap[q];
    }
    if (lane == 0) {
      s.cpre[nd] = items;
      s.tpre[nd] = tiles;
      s.total_items = items;
      s.total_tiles = tiles;
      if (blockIdx.x == 0) a.leaf_base[a.depth + 1] = lb + (int64_t)(tot >> 32);
    }
  }
  __syncthreads();
}

// smallest k with pre[k+1] > x  (pre[0] = 0, pre[n] = total)
__device__ __forceinline__ int prefix_find(const int32_t* pre, int n, int x) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// item -> (node, patch)
template <class LT>
__device__ __forceinline__ void level_item(const LevelArgs& a, const LT& s, int item,
                                           int& u, int& patch) {
  const int k = prefix_find(s.cpre, a.lvl_end - a.lvl_begin, item);
  u = a.lvl_begin + k;
  patch = a.seg_in[a.off[u] + (item - s.cpre[k])];
}

// append patch to child v's segment of the next level
template <class LT>
__device__ __forceinline__ void level_route(const PlanView& pv, const LevelArgs& a,
                                            const LT& s, int v, int patch) {
  const int slot = atomicAdd(&a.cnt[v], 1);
  const int64_t base = s.child_off[v - a.nxt_begin];
  if (pv.child_count[v] > 0) {
    a.seg_out[base + slot] = patch;
  } else {
    a.leafseg[base + slot] = patch;
    a.labels[patch] = pv.leaf_index[v];
  }
}

}  // namespace fepll
