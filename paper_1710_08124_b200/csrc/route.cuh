// Level-synchronous routing for the tree walk.
//
// The reference descends with a Python loop over the distinct nodes of each
// level (pkg/src/fepll/tree.py:416-428).  Here every level is one pass over
// the patches grouped by their current node ("segments"): a patch that picks
// child v is appended (atomic slot) to v's segment of the next level.
// Segment capacity of a child = its parent's count, so the next level's
// offsets are a prefix sum over the (at most a few hundred) nodes of the
// level, recomputed redundantly by every CTA from the final counts — no
// global scan pass.  Leaves get buckets in a separate buffer; their counts
// are the label histogram used for Wiener grouping and the cost counters.
#pragma once
#include "plan.cuh"

namespace fepll {

constexpr int kMaxLevelNodes = 1024;  // nodes per depth handled in smem

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
};

struct LevelSmem {
  int64_t pre[kMaxLevelNodes + 1];   // prefix of counts over depth-d nodes
  int64_t child_off[kMaxLevelNodes]; // offsets of depth-(d+1) nodes
  int64_t total;
};

// Every CTA: prefix over depth-d counts and the next level's segment offsets.
__device__ inline void level_setup(const PlanView& pv, const LevelArgs& a, LevelSmem& s) {
  const int nd = a.lvl_end - a.lvl_begin;
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const int u = a.lvl_begin + k;
    s.pre[k + 1] = pv.child_count[u] > 0 ? (int64_t)a.cnt[u] : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s.pre[0] = 0;
    int64_t run_int = 0, run_leaf = 0;
    const int64_t lb = a.leaf_base[a.depth];
    for (int k = 0; k < nd; ++k) {
      const int64_t c = s.pre[k + 1];
      s.pre[k + 1] = s.pre[k] + c;
      const int u = a.lvl_begin + k;
      const int nk = pv.child_count[u];
      const int cs = pv.child_start[u];
      for (int j = 0; j < nk; ++j) {
        const int v = pv.child_list[cs + j];
        if (pv.child_count[v] > 0) {
          s.child_off[v - a.nxt_begin] = run_int;
          run_int += c;
        } else {
          s.child_off[v - a.nxt_begin] = lb + run_leaf;
          run_leaf += c;
        }
      }
    }
    s.total = s.pre[nd];
    if (blockIdx.x == 0) a.leaf_base[a.depth + 1] = lb + run_leaf;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int k = threadIdx.x; k < a.nxt_end - a.nxt_begin; k += blockDim.x)
      a.off[a.nxt_begin + k] = s.child_off[k];
  }
}

// item -> (node, patch)
__device__ inline void level_item(const LevelArgs& a, const LevelSmem& s, int64_t item,
                                  int& u, int& patch) {
  int lo = 0, hi = a.lvl_end - a.lvl_begin;  // pre[lo] <= item < pre[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s.pre[mid] <= item) lo = mid; else hi = mid;
  }
  u = a.lvl_begin + lo;
  patch = a.seg_in[a.off[u] + (item - s.pre[lo])];
}

// append patch to child v's segment of the next level
__device__ inline void level_route(const PlanView& pv, const LevelArgs& a, const LevelSmem& s,
                                   int v, int patch) {
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
