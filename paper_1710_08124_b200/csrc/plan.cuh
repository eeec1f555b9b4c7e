// Device-resident plan: packed tree groups, model bases, per-beta constants,
// and the routing scratch of the level-synchronous tree walk.
#pragma once
#include <vector>

#include "common.cuh"
#include "../../include/fepll_b200.h"

namespace fepll {

// Read-only view handed to kernels by value.
struct PlanView {
  int P, n_nodes, K, T;
  const int32_t* child_start;
  const int32_t* child_count;
  const int32_t* child_list;
  const int32_t* parent;
  const int32_t* leaf_index;
  const int32_t* node_rank;
  const int32_t* grp_width;
  const int32_t* grp_col_off;
  const int32_t* child_col_off;
  const int64_t* grp_off64;
  const double* grp_basis;
  int grp_cols_total;
  const double* node_const;
  const double* node_nu_tail;
  const double* grp_sqw;
  const int32_t* model_rank;
  const int32_t* model_col_off;
  const int64_t* model_off64;
  const double* model_basis;
  int model_cols_total;
  const double* model_shrink;
  const double* model_gamma_tail;
  const float* tc_hi;
  const float* tc_lo;
  const float* tc_x;    // bf16 [lo | hi] cross-pass images (NULL if absent)
  const int64_t* tc_off;
  const int32_t* tc_npad;
  const int32_t* tc_child_col;
  const float* tc_w;
  const int32_t* tc_w_off;
  int tc_w_cols;
  int64_t tc_tstride;          // floats between consecutive iterations' B images
};

// Routing scratch: ping-pong patch-index segments per level plus the leaf
// buckets (capacity C_max * n each).
struct RouteScratch {
  int64_t cap = 0;          // patches
  int64_t seg_cap = 0;      // entries per segment buffer
  int32_t* seg[2] = {nullptr, nullptr};
  double* segsq[2] = {nullptr, nullptr};  // ||z||^2 alongside seg[] (ws2 levels read it coalesced)
  int32_t* leafseg = nullptr;
  int32_t* cnt = nullptr;     // [n_nodes] patches routed into the node this call
  int64_t* off = nullptr;     // [n_nodes] segment offset (internal: seg buf, leaf: leafseg)
  int64_t* leaf_base = nullptr;  // [levels+1]
  int32_t* queue = nullptr;   // rescore queue: (patch, node) pairs
  int32_t* queue_len = nullptr;
  int64_t queue_cap = 0;
  int32_t* node_tmp = nullptr;
  // deferred verification (plan option defer): ws2 levels route every row
  // by its tensor-core argmin and log the uncertified ones; after the last
  // level they are re-scored in FP64 and the mis-routed patches re-descended
  int4* vq = nullptr;            // (patch, node, depth, provisional child) [vq_cap]
  int64_t vq_cap = 0;
  int32_t* vq_len = nullptr;     // [2]: verify entries, repair entries
  int2* dq = nullptr;            // (patch, depth << 24 | exact child) [vq_cap]
  int32_t* first_bad = nullptr;  // [cap] earliest disagreeing depth per patch (INT_MAX-ish when none)
  int32_t* pos_leaf = nullptr;   // [cap] leafseg slot of each patch (leaf level)
  int32_t* holes = nullptr;      // [K] leaf-bucket holes per component (leaf counts subtract them)
};

// Per-plan kernel choices (fepll_plan_set_option): A/B switches between
// bitwise-equivalent kernel variants, owned by the plan so concurrent plans
// and streams never share them.
struct PlanOptions {
  int select_variant = 1;  // 0: select_ws.cu on every level, 1: select_ws2.cu, 2: ws2 on levels of <= 16 nodes
  int seg_sq = 1;          // 1: consecutive ws2 levels hand ||z||^2 over in segment order
  int wiener_pair = 1;     // 1: two 64-row CTAs per SM when they fit
  int wiener_rw = 8;       // rows per warp in the pair configuration (8 or 16)
  int wiener_xw = 0;       // 1: the Wiener kernel reads 8x8 windows of x (no Z64 rows)
  int wiener_add_dc = 1;   // 1: fepll_wiener writes est + dc; 0: the bare estimates (traces)
  int rescore_by_node = 0; // 1: re-scoring CTAs group the queued decisions by node (group matrix staged in
                           // smem once per CTA) — measured slower (select 11.3 -> 13.1 ms/step at 64 x 1024^2:
                           // one 208 KB CTA per SM leaves 8 warps for latency-bound chains), off

  int wiener_ws = 2;         // FP64 Wiener: warp-specialised kernel (12 compute + 2 loader warps, one CTA per SM; P = 64):
                             // 0 off, 1 on, 2 on from 2^20 patches (64 x 1024^2: 7.26 -> 7.06 ms/step; 8 images: 1.06 -> 1.14)
  int wiener_tc = 0;         // fepll_wiener_f32 on tcgen05 (3xTF32, wiener_tc.cu) when the shape allows; 0: FP64 DMMA
  int wiener_split = 0;      // Wiener warp pairs on 16 rows with m16n8k8 DMMAs (0: 8-row warps, m8n8k4)
  int pdl = 1;
  int defer_test = 0;        // test hook: uncertified rows routed provisionally to a wrong child
  int defer = 1;             // deferred FP64 verification of uncertified ws2 decisions (0: re-score after every level)               // tree levels and re-scoring launched with programmatic dependent launch
  int aggregate_variant = 2; // batch reprojection kernel (host: 0/1 fepll_aggregate_cover_ex, 2 fepll_aggregate_tiles)
  int l2_prefetch = 0;     // ws2 loaders prefetch rows into L2 three tiles ahead of their cp.async: 1 per 128-B line, 2 one bulk prefetch per row (both measured slower: level 0.295 -> 0.324 / 0.486 ms)
};

struct Plan {
  PlanOptions opt;
  fepll_plan_desc h{};  // sizes only (pointers are host temporaries)
  PlanView v{};
  std::vector<void*> owned;
  std::vector<int> depth;         // host copy
  std::vector<int> child_count;
  std::vector<int> level_start;   // BFS id range per depth
  std::vector<int> max_group_cols_at_depth;
  int n_levels = 0;               // depth of the deepest internal node + 1
  int max_children = 0;
  int max_inner_children = 0;     // internal children of one node
  int max_leaf_children = 0;      // leaf-bucket capacity per patch (sum over depths)
  std::vector<int> level_wide;    // per depth: a node needs the sub-group scorer
  std::vector<int> level_tc_npad; // per depth: widest tcgen05 group image
  int max_group_cols = 0;
  int max_model_rank = 0;
  int max_tc_npad = 0;
  bool have_tc = false;
  int32_t* d_leaf_nodes = nullptr;   // BFS ids of the leaves, ascending
  int n_leaf_nodes = 0;
  RouteScratch rs;
  uint8_t* wtc_img = nullptr;        // tcgen05 Wiener basis images (wiener_tc.cu), owned
  int last_n_total = 0;
  // optional timing of the level kernels (fepll_plan_profile): event pairs
  std::vector<cudaEvent_t> prof_ev;
  int prof_used = 0;
};

}  // namespace fepll
