// Plan lifetime: upload of the packed tree/model and routing scratch.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>

#include "plan.cuh"

namespace fepll {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};
void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

template <typename T>
static int upload(Plan* p, const T* src, int64_t count, const T** dst) {
  if (count <= 0 || src == nullptr) {
    *dst = nullptr;
    return kOk;
  }
  void* d = nullptr;
  FEPLL_CUDA(cudaMalloc(&d, sizeof(T) * count));
  p->owned.push_back(d);
  FEPLL_CUDA(cudaMemcpy(d, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  *dst = static_cast<const T*>(d);
  return kOk;
}

#define UP(src, count, dst)                                  \
  do {                                                       \
    int _rc = upload(p, (src), (int64_t)(count), &(dst));    \
    if (_rc) return _rc;                                     \
  } while (0)

int wiener_tc_prepare(Plan* p);  // wiener_tc.cu

static int create(const fepll_plan_desc* d, Plan** out) {
  FEPLL_REQUIRE(d != nullptr && out != nullptr, "null plan descriptor");
  FEPLL_REQUIRE(d->patch_dim > 0 && d->patch_dim <= kMaxP, "patch_dim out of range (1..256)");
  FEPLL_REQUIRE(d->n_nodes >= 1 && d->n_components >= 1 && d->iterations >= 1, "empty plan");
  Plan* p = new Plan();
  p->h = *d;
  const int n = d->n_nodes, K = d->n_components, T = d->iterations;
  PlanView& v = p->v;
  v.P = d->patch_dim;
  v.n_nodes = n;
  v.K = K;
  v.T = T;
  v.grp_cols_total = d->grp_cols_total;
  v.model_cols_total = d->model_cols_total;
  p->depth.assign(d->depth, d->depth + n);
  p->child_count.assign(d->child_count, d->child_count + n);
  int maxd = 0;
  for (int i = 0; i < n; ++i) {
    maxd = std::max(maxd, d->depth[i]);
    if (i && d->depth[i] < d->depth[i - 1]) {
      set_error("nodes are not in BFS (depth-sorted) order");
      delete p;
      return kDataError;
    }
    p->max_children = std::max(p->max_children, d->child_count[i]);
    p->max_group_cols = std::max(p->max_group_cols, d->grp_width[i]);
  }
  for (int k = 0; k < K; ++k) p->max_model_rank = std::max(p->max_model_rank, d->model_rank[k]);
  // segment capacities: a child's segment holds up to its parent's count
  // (leaf buckets of every depth share one array: sum the per-depth maxima)
  {
    std::vector<int> leaf_at_depth(maxd + 1, 0);
    for (int u = 0; u < n; ++u) {
      int inner = 0, leaves = 0;
      for (int j = 0; j < d->child_count[u]; ++j)
        (d->child_count[d->child_list[d->child_start[u] + j]] > 0 ? inner : leaves) += 1;
      p->max_inner_children = std::max(p->max_inner_children, inner);
      leaf_at_depth[d->depth[u]] = std::max(leaf_at_depth[d->depth[u]], leaves);
    }
    for (int x : leaf_at_depth) p->max_leaf_children += x;
  }
  p->level_start.assign(maxd + 2, 0);
  for (int dd = 0, i = 0; dd <= maxd + 1; ++dd) {
    while (i < n && d->depth[i] < dd) ++i;
    p->level_start[dd] = i;
  }
  if (maxd + 1 >= kMaxDepth) {
    set_error("tree deeper than 62 levels");
    delete p;
    return kDataError;
  }
  for (int dd = 0; dd <= maxd; ++dd) {
    if (p->level_start[dd + 1] - p->level_start[dd] > 512) {
      set_error("a tree level holds more than 512 nodes");
      delete p;
      return kDataError;
    }
  }
  p->n_levels = 0;
  for (int i = 0; i < n; ++i)
    if (d->child_count[i] > 0) p->n_levels = std::max(p->n_levels, d->depth[i] + 1);
  // "wide" levels hold a node beyond the single-pass scorers' limits (more
  // than 32 children or 512 group columns — e.g. the exhaustive star tree);
  // they are scored in sub-groups / column chunks
  p->level_wide.assign(maxd + 1, 0);
  p->level_tc_npad.assign(maxd + 1, 0);
  p->max_group_cols_at_depth.assign(maxd + 1, 0);
  for (int i = 0; i < n; ++i) {
    p->max_group_cols_at_depth[d->depth[i]] = std::max(p->max_group_cols_at_depth[d->depth[i]], d->grp_width[i]);
    if (d->child_count[i] > kMaxChildren || d->grp_width[i] > kMaxGroupCols) p->level_wide[d->depth[i]] = 1;
    if (d->grp_tc_npad)
      p->level_tc_npad[d->depth[i]] = std::max(p->level_tc_npad[d->depth[i]], d->grp_tc_npad[i]);
  }
  UP(d->child_start, n, v.child_start);
  UP(d->child_count, n, v.child_count);
  UP(d->child_list, std::max(n - 1, 1), v.child_list);
  UP(d->leaf_index, n, v.leaf_index);
  {
    std::vector<int32_t> parent(n, 0);
    for (int u = 0; u < n; ++u)
      for (int j = 0; j < d->child_count[u]; ++j) parent[d->child_list[d->child_start[u] + j]] = u;
    UP(parent.data(), n, v.parent);
  }
  UP(d->node_rank, n, v.node_rank);
  UP(d->grp_width, n, v.grp_width);
  UP(d->grp_col_off, n, v.grp_col_off);
  UP(d->child_col_off, n, v.child_col_off);
  UP(d->grp_off64, n, v.grp_off64);
  UP(d->grp_basis, d->grp_basis_len, v.grp_basis);
  UP(d->node_const, (int64_t)T * n, v.node_const);
  UP(d->node_nu_tail, (int64_t)T * n, v.node_nu_tail);
  UP(d->grp_sqw, (int64_t)T * d->grp_cols_total, v.grp_sqw);
  UP(d->model_rank, K, v.model_rank);
  UP(d->model_col_off, K, v.model_col_off);
  UP(d->model_off64, K, v.model_off64);
  UP(d->model_basis, d->model_basis_len, v.model_basis);
  UP(d->model_shrink, (int64_t)T * d->model_cols_total, v.model_shrink);
  UP(d->model_gamma_tail, (int64_t)T * K, v.model_gamma_tail);
  if (d->grp_tc_hi && d->grp_tc_lo && d->grp_tc_len > 0) {
    UP(d->grp_tc_hi, d->grp_tc_len, v.tc_hi);
    UP(d->grp_tc_lo, d->grp_tc_len, v.tc_lo);
    if (d->grp_tc_x) UP(d->grp_tc_x, d->grp_tc_len, v.tc_x);
    UP(d->grp_tc_off, n, v.tc_off);
    UP(d->grp_tc_npad, n, v.tc_npad);
    UP(d->grp_tc_child_col, n, v.tc_child_col);
    UP(d->grp_tc_w, (int64_t)T * d->grp_tc_w_cols, v.tc_w);
    UP(d->grp_tc_w_off, n, v.tc_w_off);
    v.tc_w_cols = d->grp_tc_w_cols;
    FEPLL_REQUIRE(d->grp_tc_len % T == 0, "plan: tcgen05 images must hold one block per iteration");
    v.tc_tstride = d->grp_tc_len / T;
    p->have_tc = true;
    for (int i = 0; i < n; ++i) p->max_tc_npad = std::max(p->max_tc_npad, d->grp_tc_npad[i]);
  }
  {
    std::vector<int32_t> leaves;
    for (int i = 0; i < n; ++i)
      if (d->child_count[i] == 0) leaves.push_back(i);
    p->n_leaf_nodes = (int)leaves.size();
    const int32_t* dl = nullptr;
    UP(leaves.data(), leaves.size(), dl);
    p->d_leaf_nodes = const_cast<int32_t*>(dl);
  }
  // per-node scratch
  void* m = nullptr;
  FEPLL_CUDA(cudaMalloc(&m, sizeof(int32_t) * n));
  p->owned.push_back(m);
  p->rs.cnt = static_cast<int32_t*>(m);
  FEPLL_CUDA(cudaMalloc(&m, sizeof(int64_t) * n));
  p->owned.push_back(m);
  p->rs.off = static_cast<int64_t*>(m);
  FEPLL_CUDA(cudaMalloc(&m, sizeof(int64_t) * (maxd + 3)));
  p->owned.push_back(m);
  p->rs.leaf_base = static_cast<int64_t*>(m);
  FEPLL_CUDA(cudaMalloc(&m, sizeof(int32_t) * kMaxDepth));
  p->owned.push_back(m);
  p->rs.queue_len = static_cast<int32_t*>(m);
  FEPLL_CUDA(cudaMalloc(&m, sizeof(int32_t) * 2));
  p->owned.push_back(m);
  p->rs.vq_len = static_cast<int32_t*>(m);
  FEPLL_CUDA(cudaMalloc(&m, sizeof(int32_t) * std::max(1, p->v.K)));
  p->owned.push_back(m);
  p->rs.holes = static_cast<int32_t*>(m);
  {
    const int rc = wiener_tc_prepare(p);
    if (rc) return rc;
  }
  *out = p;
  return kOk;
}

static void free_scratch(Plan* p) {
  RouteScratch& r = p->rs;
  cudaFree(r.seg[0]);
  cudaFree(r.seg[1]);
  cudaFree(r.segsq[0]);
  cudaFree(r.segsq[1]);
  r.segsq[0] = r.segsq[1] = nullptr;
  cudaFree(r.leafseg);
  cudaFree(r.queue);
  cudaFree(r.vq);
  cudaFree(r.dq);
  cudaFree(r.first_bad);
  cudaFree(r.pos_leaf);
  r.seg[0] = r.seg[1] = r.leafseg = r.queue = nullptr;
  r.vq = nullptr;
  r.dq = nullptr;
  r.first_bad = r.pos_leaf = nullptr;
  r.cap = r.seg_cap = r.queue_cap = r.vq_cap = 0;
}

static int reserve(Plan* p, int64_t max_patches) {
  FEPLL_REQUIRE(max_patches >= 0 && max_patches < (int64_t(1) << 31), "patch count out of range");
  if (max_patches <= p->rs.cap) return kOk;
  free_scratch(p);
  RouteScratch& r = p->rs;
  const int64_t np = std::max<int64_t>(1, max_patches);
  const int64_t seg = np * std::max(1, p->max_inner_children);
  const int64_t lseg = np * std::max(1, p->max_leaf_children);
  FEPLL_CUDA(cudaMalloc(&r.seg[0], sizeof(int32_t) * std::max(seg, np)));  // level 0 = all patches
  FEPLL_CUDA(cudaMalloc(&r.seg[1], sizeof(int32_t) * seg));
  FEPLL_CUDA(cudaMalloc(&r.segsq[0], sizeof(double) * std::max(seg, np)));
  FEPLL_CUDA(cudaMalloc(&r.segsq[1], sizeof(double) * seg));
  // leaf buckets: capacity = leaf_capacity(the parent's count) (route.cuh),
  // room for patches re-routed by the deferred verification
  FEPLL_CUDA(cudaMalloc(&r.leafseg, sizeof(int32_t) * (lseg + lseg / 4 + (int64_t)kLeafSlack * std::max(1, p->v.K))));
  r.queue_cap = std::max<int64_t>(1024, max_patches);
  FEPLL_CUDA(cudaMalloc(&r.queue, sizeof(int32_t) * 2 * r.queue_cap));
  // every patch can be logged once per level
  r.vq_cap = std::max<int64_t>(1024, np * std::max(1, p->n_levels));
  FEPLL_CUDA(cudaMalloc(&r.vq, sizeof(int4) * r.vq_cap));
  FEPLL_CUDA(cudaMalloc(&r.dq, sizeof(int2) * r.vq_cap));
  FEPLL_CUDA(cudaMalloc(&r.first_bad, sizeof(int32_t) * np));
  FEPLL_CUDA(cudaMemset(r.first_bad, 0x7f, sizeof(int32_t) * np));
  FEPLL_CUDA(cudaMalloc(&r.pos_leaf, sizeof(int32_t) * np));
  r.cap = max_patches;
  r.seg_cap = seg;
  return kOk;
}

}  // namespace fepll

using fepll::Plan;

extern "C" {

int fepll_abi_version(void) { return 1; }

int64_t fepll_launch_count(void) { return fepll::g_launches.load(); }

const char* fepll_last_error(void) { return fepll::g_last_error.c_str(); }

int fepll_plan_create(const fepll_plan_desc* desc, fepll_plan_t* out) {
  Plan* p = nullptr;
  int rc = fepll::create(desc, &p);
  if (rc) return rc;
  *out = reinterpret_cast<fepll_plan_t>(p);
  return fepll::kOk;
}

int fepll_plan_reserve(fepll_plan_t plan, int64_t max_patches) {
  return fepll::reserve(reinterpret_cast<Plan*>(plan), max_patches);
}

int fepll_plan_profile(fepll_plan_t plan, int32_t capacity) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && capacity >= 0, "plan_profile: bad arguments");
  for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
  p->prof_ev.assign(2 * (size_t)capacity, nullptr);
  for (auto& e : p->prof_ev) FEPLL_CUDA(cudaEventCreate(&e));
  p->prof_used = 0;
  return fepll::kOk;
}

int fepll_plan_profile_read(fepll_plan_t plan, double* total_ms, int32_t* launches) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && total_ms && launches, "plan_profile_read: bad arguments");
  double sum = 0.0;
  if (p->prof_used > 0) FEPLL_CUDA(cudaEventSynchronize(p->prof_ev[2 * p->prof_used - 1]));
  for (int i = 0; i < p->prof_used; ++i) {
    float ms = 0.f;
    FEPLL_CUDA(cudaEventElapsedTime(&ms, p->prof_ev[2 * i], p->prof_ev[2 * i + 1]));
    sum += ms;
  }
  *total_ms = sum;
  *launches = p->prof_used;
  p->prof_used = 0;
  return fepll::kOk;
}

static int* plan_option(Plan* p, const char* name) {
  const std::string n(name ? name : "");
  if (n == "select_variant") return &p->opt.select_variant;
  if (n == "seg_sq") return &p->opt.seg_sq;
  if (n == "wiener_pair") return &p->opt.wiener_pair;
  if (n == "wiener_rw") return &p->opt.wiener_rw;
  if (n == "wiener_xw") return &p->opt.wiener_xw;
  if (n == "wiener_add_dc") return &p->opt.wiener_add_dc;
  if (n == "l2_prefetch") return &p->opt.l2_prefetch;
  if (n == "rescore_by_node") return &p->opt.rescore_by_node;
  if (n == "aggregate_variant") return &p->opt.aggregate_variant;
  if (n == "pdl") return &p->opt.pdl;
  if (n == "defer") return &p->opt.defer;
  if (n == "defer_test") return &p->opt.defer_test;
  if (n == "wiener_split") return &p->opt.wiener_split;
  if (n == "wiener_tc") return &p->opt.wiener_tc;
  if (n == "wiener_ws") return &p->opt.wiener_ws;
  return nullptr;
}

int fepll_plan_set_option(fepll_plan_t plan, const char* name, int64_t value) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr, "plan_set_option: bad arguments");
  int* slot = plan_option(p, name);
  FEPLL_REQUIRE(slot != nullptr, std::string("plan_set_option: unknown option ") + (name ? name : "(null)"));
  const std::string n(name);
  const bool ok = (n == "select_variant" || n == "l2_prefetch" || n == "aggregate_variant" || n == "wiener_ws")
                      ? (value >= 0 && value <= 2)
                  : (n == "wiener_rw")    ? (value == 8 || value == 16)
                                          : (value == 0 || value == 1);
  FEPLL_REQUIRE(ok, "plan_set_option: value out of range for " + n);
  *slot = (int)value;
  return fepll::kOk;
}

int fepll_plan_get_option(fepll_plan_t plan, const char* name, int64_t* value) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  FEPLL_REQUIRE(p != nullptr && value != nullptr, "plan_get_option: bad arguments");
  int* slot = plan_option(p, name);
  FEPLL_REQUIRE(slot != nullptr, std::string("plan_get_option: unknown option ") + (name ? name : "(null)"));
  *value = *slot;
  return fepll::kOk;
}

namespace {
__global__ void stamp_kernel(uint64_t* dst) {
  uint64_t g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  *dst = g;
}
}  // namespace

int fepll_stamp(uint64_t* dst, void* stream) {
  FEPLL_REQUIRE(dst != nullptr, "stamp: bad arguments");
  stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(dst);
  FEPLL_LAUNCH();
  return fepll::kOk;
}

int fepll_plan_destroy(fepll_plan_t plan) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return fepll::kOk;
  for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
  fepll::free_scratch(p);
  for (void* m : p->owned) cudaFree(m);
  delete p;
  return fepll::kOk;
}

}  // extern "C"
