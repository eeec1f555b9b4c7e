// Kernel (b), tensor-core path: one tree level as a grouped GEMM on tcgen05.
//
// Restates the per-level work of pkg/src/fepll/tree.py:416-428 (score all
// children of the current node, first-minimum child wins) with the score of
// pkg/src/fepll/gmm.py:323-339.  Patches of one level are grouped by node
// (route.cuh); a tile is 128 patches of one node.  For a tile:
//
//   C (128 x N) = Z_tile (128 x P) . G_u (P x N)     N = sum of child ranks
//
// runs as 3xTF32 on tcgen05 (kind::tf32, M=128, K=8 per MMA, FP32 accumulator
// in TMEM): D = Zhi.Ghi + Zhi.Glo + Zlo.Ghi.  Operands are K-major,
// 128-byte-swizzled: the group image G_u arrives pre-split/pre-swizzled by
// the TMA bulk engine, the patch rows are gathered by the CTA's threads,
// split hi/lo and stored swizzled.  The K dimension streams through two
// smem stages (one 32-float K atom each) so loads overlap the MMAs.
//
// Epilogue (one thread per patch row, TMEM lane == row): FP64
// sum_j c_j^2 w_j per child, score, argmin, and an error bound
// err_c = guard * ||z|| * sum_j |c_j w_j| on each score (the 3xTF32
// projection error is <= guard/2 * ||z|| per coefficient).  A decision whose
// runner-up lies within err_best + err_runner is not taken here: the patch
// is queued for exact FP64 re-scoring (select.cu), so the chosen child always
// equals the FP64 argmin.
#include "route.cuh"
#include "tc.cuh"
#include "tc_epi.cuh"

namespace fepll {

constexpr int kTcRows = 128;          // M
constexpr int kTcThreads = 128;       // 4 warps: loaders + epilogue; thread 0 issues MMAs
constexpr int kAtomFloats = 32;       // 128-byte K atom
constexpr int kAtomBytesA = kTcRows * 128;
constexpr uint32_t kTmemCols = 256;   // one accumulator, N <= 256

struct TcSmemTables {
  LevelTables lv;
  EpiChild ch;
  int32_t rows[kTcRows];
  int32_t key[kTcRows];
  int32_t lrank[kTcRows];
  int32_t lrank2[kTcRows];  // deferred verification: the row's log slot
  int32_t bcnt[kMaxChildren + 1];
  int32_t bbase[kMaxChildren + 1];
  uint64_t mma_bar[2];
  uint64_t load_bar[2];
  uint32_t tmem_base;
};

struct TcArgs {
  LevelArgs a;
  const float* Z32;
  int z32_pitch;
  const double* sq;
  double guard;
  int32_t* queue;
  int32_t* queue_len;  // [depth]
  // deferred verification (vq != NULL, select.cu): uncertified rows are
  // routed by the tensor-core argmin and logged
  int4* vq;
  int32_t* vq_len;
  int64_t vq_cap;
  int32_t* pos_leaf;
  int perturb;         // test hook (plan option defer_test): uncertified rows take the next child
  int katoms;
  int bmax_rows;       // padded N of the stage buffers
};

__global__ void __launch_bounds__(kTcThreads, 1)
select_level_tc_kernel(PlanView pv, TcArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the operand region (SWIZZLE_128B atoms)
  uint8_t* base = tc::align1024(smem_raw);
  const int bstage = args.bmax_rows * 128;               // bytes of one B half per stage
  const int stage_bytes = 2 * kAtomBytesA + 2 * bstage;
  TcSmemTables& s = *reinterpret_cast<TcSmemTables*>(base + 2 * stage_bytes);
  const LevelArgs& a = args.a;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (warp == 0) tc::tmem_alloc(&s.tmem_base, kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.mma_bar[i], 1);
      tc::mbar_init(&s.load_bar[i], 1);
    }
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s.tmem_base;
  // levels of <= 256 nodes on both sides: the one-warp tables (one barrier), else the block scans
  if (a.lvl_end - a.lvl_begin <= 256 && a.nxt_end - a.nxt_begin <= 256) level_tables_warp(pv, a, s.lv, kTcRows);
  else level_tables(pv, a, s.lv, kTcRows);

  const int nd = a.lvl_end - a.lvl_begin;
  const int t = a.t;
  uint32_t uses[2] = {0, 0};  // completed-or-pending commits per stage (uniform across threads)
  const double guard = args.guard;

  for (int tile = blockIdx.x; tile < s.lv.total_tiles; tile += gridDim.x) {
    // tile -> node, row range
    const int lo = prefix_find(s.lv.tpre, nd, tile);
    const int u = a.lvl_begin + lo;
    const int first = (tile - s.lv.tpre[lo]) * kTcRows;
    const int cnt_u = s.lv.cpre[lo + 1] - s.lv.cpre[lo];
    const int m = min(kTcRows, cnt_u - first);
    const int npad = pv.tc_npad[u];
    const int nk = pv.child_count[u];
    const int64_t seg0 = a.off[u] + first;
    // per-tile tables (previous tile's epilogue finished: trailing __syncthreads)
    epi_load_node(pv, t, u, s.ch, tid, kTcThreads);
    const int my_patch = tid < m ? a.seg_in[seg0 + tid] : -1;
    s.rows[tid] = my_patch;
    const float* zrow = my_patch >= 0 ? args.Z32 + (int64_t)my_patch * args.z32_pitch : nullptr;
    const float* bhi = pv.tc_hi + (int64_t)t * pv.tc_tstride + pv.tc_off[u];
    const float* blo = pv.tc_lo + (int64_t)t * pv.tc_tstride + pv.tc_off[u];
    const uint32_t bbytes = (uint32_t)npad * 128u;
    const uint32_t idesc = tc::idesc_tf32(kTcRows, npad);

    int last_stage = 0;
    for (int ka = 0; ka < args.katoms; ++ka) {
      const int st = ka & 1;  // stage parity alternates within and across tiles via uses[]
      // the stage is free once the MMAs that last read it have completed
      if (uses[st] > 0) tc::mbar_wait(&s.mma_bar[st], (uses[st] - 1) & 1);
      uint8_t* sA_hi = base + st * stage_bytes;
      uint8_t* sA_lo = sA_hi + kAtomBytesA;
      uint8_t* sB_hi = sA_lo + kAtomBytesA;
      uint8_t* sB_lo = sB_hi + bstage;
      if (tid == 0) {
        tc::mbar_arrive_expect_tx(&s.load_bar[st], 2 * bbytes);
        tc::bulk_g2s(sB_hi, bhi + (int64_t)ka * npad * kAtomFloats, bbytes, &s.load_bar[st]);
        tc::bulk_g2s(sB_lo, blo + (int64_t)ka * npad * kAtomFloats, bbytes, &s.load_bar[st]);
      }
      // A atom: row tid, 8 chunks of 16 B, chunk c stored at c ^ (row % 8)
      {
        const int r8 = tid & 7;
        uint8_t* dhi = sA_hi + (tid >> 3) * 1024 + r8 * 128;
        uint8_t* dlo = sA_lo + (tid >> 3) * 1024 + r8 * 128;
        const float4* src = zrow ? reinterpret_cast<const float4*>(zrow + ka * kAtomFloats) : nullptr;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 v = src ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          float4 h, l;
          h.x = tc::to_tf32(v.x); l.x = v.x - h.x;
          h.y = tc::to_tf32(v.y); l.y = v.y - h.y;
          h.z = tc::to_tf32(v.z); l.z = v.z - h.z;
          h.w = tc::to_tf32(v.w); l.w = v.w - h.w;
          *reinterpret_cast<float4*>(dhi + ((c ^ r8) << 4)) = h;
          *reinterpret_cast<float4*>(dlo + ((c ^ r8) << 4)) = l;
        }
      }
      tc::fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::mbar_wait(&s.load_bar[st], uses[st] & 1);
        tc::fence_after_sync();
        const uint32_t a_hi = tc::smem_u32(sA_hi), a_lo = tc::smem_u32(sA_lo);
        const uint32_t b_hi = tc::smem_u32(sB_hi), b_lo = tc::smem_u32(sB_lo);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t ko = kk * 32;  // 8 tf32 = 32 bytes inside the swizzle atom
          const uint32_t acc = (ka > 0 || kk > 0) ? 1u : 0u;
          tc::mma_tf32(tmem, tc::desc_sw128(a_hi + ko), tc::desc_sw128(b_hi + ko), idesc, acc);
          tc::mma_tf32(tmem, tc::desc_sw128(a_hi + ko), tc::desc_sw128(b_lo + ko), idesc, 1u);
          tc::mma_tf32(tmem, tc::desc_sw128(a_lo + ko), tc::desc_sw128(b_hi + ko), idesc, 1u);
        }
        tc::mma_commit(&s.mma_bar[st]);
      }
      uses[st] += 1;
      last_stage = st;
    }
    // accumulators complete
    tc::mbar_wait(&s.mma_bar[last_stage], (uses[last_stage] - 1) & 1);
    tc::fence_after_sync();

    // ---- epilogue: thread tid owns TMEM lane tid == tile row tid
    const bool valid = tid < m;
    const double sqv = valid ? args.sq[my_patch] : 0.0;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    bool flagged;
    int bi = epi_score_row(s.ch, nk, lane_base, sqv, guard, &flagged);
    if (args.vq && args.perturb && flagged && nk > 1) bi = bi + 1 < nk ? bi + 1 : 0;  // test hook
    // ---- routing (aggregated per tile: one global atomic per child)
    tc::fence_before_sync();
    if (tid <= kMaxChildren) s.bcnt[tid] = 0;
    __syncthreads();
    const bool defer = args.vq != nullptr;
    if (valid) {
      const int key = (flagged && !defer) ? kMaxChildren : bi;
      s.key[tid] = key;
      s.lrank[tid] = atomicAdd(&s.bcnt[key], 1);
      if (defer && flagged) s.lrank2[tid] = atomicAdd(&s.bcnt[kMaxChildren], 1);
    }
    __syncthreads();
    if (tid < nk && s.bcnt[tid] > 0) s.bbase[tid] = atomicAdd(&a.cnt[s.ch.bfs[tid]], s.bcnt[tid]);
    if (tid == kTcThreads - 1 && s.bcnt[kMaxChildren] > 0) {
      if (defer) {
        s.bbase[kMaxChildren] = atomicAdd(args.vq_len, s.bcnt[kMaxChildren]);
        atomicAdd(&args.queue_len[a.depth], s.bcnt[kMaxChildren]);  // per-level statistics
      } else {
        s.bbase[kMaxChildren] = atomicAdd(&args.queue_len[a.depth], s.bcnt[kMaxChildren]);
      }
    }
    __syncthreads();
    if (valid) {
      const int key = s.key[tid];
      const int slot = s.bbase[key] + s.lrank[tid];
      if (key == kMaxChildren) {
        args.queue[2 * slot] = my_patch;
        args.queue[2 * slot + 1] = u;
      } else {
        const int v = s.ch.bfs[key];
        const int64_t b0 = s.lv.child_off[v - a.nxt_begin];
        if (pv.child_count[v] > 0) {
          a.seg_out[b0 + slot] = my_patch;
        } else {
          a.leafseg[b0 + slot] = my_patch;
          a.labels[my_patch] = pv.leaf_index[v];
          if (defer) args.pos_leaf[my_patch] = (int32_t)(b0 + slot);
        }
        if (defer && flagged) {  // the provisional decision, verified after the last level
          const int64_t s2 = (int64_t)s.bbase[kMaxChildren] + s.lrank2[tid];
          if (s2 < args.vq_cap) args.vq[s2] = make_int4(my_patch, u, a.depth, v);
          else atomicOr(&args.queue_len[kMaxDepth - 1], 1);
        }
      }
    }
    __syncthreads();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kTmemCols);
}

static size_t tc_smem_bytes(int bmax_rows) {
  const size_t stage = 2 * (size_t)kAtomBytesA + 2 * (size_t)bmax_rows * 128;
  return 1024 + 2 * stage + sizeof(TcSmemTables);
}

bool deferred_verify(const Plan* p);

int select_level_tc(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                    cudaStream_t st) {
  FEPLL_REQUIRE(!p->level_wide[a.depth] && p->level_tc_npad[a.depth] <= 256,
                "tensor level kernel: node wider than 256 padded columns");
  const int P = p->v.P;
  const int ppad = (P + 31) / 32 * 32;
  const int bmax = std::max(16, p->level_tc_npad[a.depth]);
  TcArgs args;
  args.a = a;
  args.Z32 = Z32;
  args.z32_pitch = ppad;
  args.sq = sq;
  args.guard = guard > 0 ? guard : kDefaultGuard;
  args.queue = p->rs.queue;
  args.queue_len = p->rs.queue_len;
  args.vq = deferred_verify(p) ? p->rs.vq : nullptr;
  args.vq_len = p->rs.vq_len;
  args.vq_cap = p->rs.vq_cap;
  args.pos_leaf = p->rs.pos_leaf;
  args.perturb = p->opt.defer_test;
  args.katoms = ppad / 32;
  args.bmax_rows = bmax;
  const size_t smem = tc_smem_bytes(bmax);
  FEPLL_CUDA(cudaFuncSetAttribute(select_level_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  select_level_tc_kernel<<<kSMs, kTcThreads, smem, st>>>(p->v, args);
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll
