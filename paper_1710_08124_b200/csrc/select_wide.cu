// Kernel (b), tensor-core path for wide nodes: the exhaustive scan of
// pkg/src/fepll/gmm.py:371-391 (select_exhaustive — argmin over all K
// components, lowest index on ties), run as the one-level star tree of
// tree.star_tree, and any node beyond the single-pass limits (> 32 children
// or > 256 padded columns).
//
// A tile is 128 patches of one node.  Its TF32 hi/lo rows stay resident in
// shared memory while the node's group image streams through in column
// chunks (consecutive children, <= NW padded columns, <= 32 children): per
// chunk, 3xTF32 tcgen05 MMAs (B chunk per K atom by TMA bulk copies, double
// buffered) into a TMEM accumulator, then the per-row epilogue folds the
// chunk's children into a running certified argmin (tc_epi.cuh EpiRun).
// Uncertified rows go to the FP64 re-scoring queue as in select_tc.cu, so
// the chosen component is the FP64 argmin.  The exhaustive scan is a plain
// GEMM Z (n x P) . U_all (P x sum r_k) with a segmented argmin — this is
// its tensor-core form.
#include "route.cuh"
#include "tc.cuh"
#include "tc_epi.cuh"

namespace fepll {

namespace wide {

constexpr int kRows = 128;
constexpr int kThreads = 128;
constexpr int kAtomBytes = kRows * 128;  // one K atom of A (hi or lo)
constexpr uint32_t kTmemCols = 256;

struct Tables {
  LevelTables lv;
  EpiChild ch;
  uint64_t mma_bar[2];
  uint64_t load_bar[2];
  uint64_t done_bar;
  uint32_t tmem_base;
};

struct Args {
  LevelArgs a;
  const float* Z32;
  int z32_pitch;
  const double* sq;
  double guard;
  int32_t* queue;
  int32_t* queue_len;
  int katoms;
  int nw;  // max padded columns per chunk (<= 256)
};

__global__ void __launch_bounds__(kThreads, 1)
select_level_wide_kernel(PlanView pv, Args args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = tc::align1024(smem_raw);
  uint8_t* A = base;                                          // [katoms][hi, lo][128 rows]
  uint8_t* Bst = A + 2 * args.katoms * kAtomBytes;            // [2 stages][hi, lo][nw rows]
  const int bhalf = args.nw * 128;
  Tables& s = *reinterpret_cast<Tables*>(Bst + 2 * 2 * bhalf);
  const LevelArgs& a = args.a;
  const int tid = threadIdx.x, warp = tid >> 5;

  if (warp == 0) tc::tmem_alloc(&s.tmem_base, kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.mma_bar[i], 1);
      tc::mbar_init(&s.load_bar[i], 1);
    }
    tc::mbar_init(&s.done_bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s.tmem_base;
  level_tables(pv, a, s.lv, kRows);
  const int nd = a.lvl_end - a.lvl_begin;
  const int t = a.t;
  uint32_t uses[2] = {0, 0};  // commits per B stage (uniform)
  uint32_t dones = 0;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);

  for (int tile = blockIdx.x; tile < s.lv.total_tiles; tile += gridDim.x) {
    const int lo = prefix_find(s.lv.tpre, nd, tile);
    const int u = a.lvl_begin + lo;
    const int first = (tile - s.lv.tpre[lo]) * kRows;
    const int m = min(kRows, (s.lv.cpre[lo + 1] - s.lv.cpre[lo]) - first);
    const int nk = pv.child_count[u];
    const int npad = pv.tc_npad[u];
    const int32_t* kids = pv.child_list + pv.child_start[u];
    const int my_patch = tid < m ? a.seg_in[a.off[u] + first + tid] : -1;
    // ---- A: this tile's rows, TF32 hi/lo split, 128B-swizzled, all K atoms
    {
      const int r8 = tid & 7;
      const float* zrow = my_patch >= 0 ? args.Z32 + (int64_t)my_patch * args.z32_pitch : nullptr;
      for (int ka = 0; ka < args.katoms; ++ka) {
        uint8_t* dhi = A + (2 * ka) * kAtomBytes + (tid >> 3) * 1024 + r8 * 128;
        uint8_t* dlo = A + (2 * ka + 1) * kAtomBytes + (tid >> 3) * 1024 + r8 * 128;
        const float4* src = zrow ? reinterpret_cast<const float4*>(zrow + ka * 32) : nullptr;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = src ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
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
    }
    const double sqv = my_patch >= 0 ? args.sq[my_patch] : 0.0;
    EpiRun run;
    // ---- column chunks of consecutive children
    for (int k0 = 0; k0 < nk;) {
      const int col0 = pv.tc_child_col[kids[k0]];
      int k1 = k0, width = 0;
      while (k1 < nk && k1 - k0 < kMaxChildren) {
        const int v = kids[k1];
        const int end = pv.tc_child_col[v] + ((pv.node_rank[v] + 15) & ~15) - col0;
        if (end > args.nw) break;
        width = end;
        ++k1;
      }
      const int nkc = k1 - k0;
      __syncthreads();  // previous chunk's epilogue is done with the tables and TMEM
      // chunk tables: children k0..k1-1 relative to col0
      {
        const float* w = pv.tc_w + (int64_t)t * pv.tc_w_cols + pv.tc_w_off[u] + col0;
        for (int j = tid; j < width; j += kThreads) s.ch.w[j] = w[j];
        if (tid < nkc) {
          const int v = kids[k0 + tid];
          const int64_t ti = (int64_t)t * pv.n_nodes + v;
          s.ch.cconst[tid] = pv.node_const[ti];
          s.ch.cinvnut[tid] = 1.0 / pv.node_nu_tail[ti];
          const float* wc = w + (pv.tc_child_col[v] - col0);
          double n2 = 0.0;
          for (int j = 0; j < pv.node_rank[v]; ++j) n2 += (double)wc[j] * (double)wc[j];
          s.ch.wnorm[tid] = sqrt(n2);
          s.ch.col[tid] = pv.tc_child_col[v] - col0;
          s.ch.chunks[tid] = (pv.node_rank[v] + 15) >> 4;
          s.ch.bfs[tid] = v;
        }
      }
      tc::fence_before_sync();
      __syncthreads();
      tc::fence_after_sync();
      if (tid == 0) {
        const uint32_t idesc = tc::idesc_tf32(kRows, width);
        const uint32_t bbytes = (uint32_t)width * 128u;
        for (int ka = 0; ka < args.katoms; ++ka) {
          const int st = ka & 1;
          if (uses[st] > 0) tc::mbar_wait(&s.mma_bar[st], (uses[st] - 1) & 1);
          uint8_t* bhi = Bst + st * 2 * bhalf;
          uint8_t* blo = bhi + bhalf;
          // rows [col0, col0 + width) of atom ka: contiguous 128-byte rows, 16-row aligned
          const int64_t off = (int64_t)t * pv.tc_tstride + pv.tc_off[u] + ((int64_t)ka * npad + col0) * 32;
          tc::mbar_arrive_expect_tx(&s.load_bar[st], 2 * bbytes);
          tc::bulk_g2s(bhi, pv.tc_hi + off, bbytes, &s.load_bar[st]);
          tc::bulk_g2s(blo, pv.tc_lo + off, bbytes, &s.load_bar[st]);
          tc::mbar_wait(&s.load_bar[st], uses[st] & 1);
          tc::fence_after_sync();
          const uint32_t a_hi = tc::smem_u32(A + (2 * ka) * kAtomBytes);
          const uint32_t a_lo = tc::smem_u32(A + (2 * ka + 1) * kAtomBytes);
          const uint32_t b_hi = tc::smem_u32(bhi), b_lo = tc::smem_u32(blo);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t ko = kk * 32;
            const uint32_t acc = (ka > 0 || kk > 0) ? 1u : 0u;
            tc::mma_tf32(tmem, tc::desc_sw128(a_lo + ko), tc::desc_sw128(b_hi + ko), idesc, acc);
            tc::mma_tf32(tmem, tc::desc_sw128(a_hi + ko), tc::desc_sw128(b_lo + ko), idesc, 1u);
            tc::mma_tf32(tmem, tc::desc_sw128(a_hi + ko), tc::desc_sw128(b_hi + ko), idesc, 1u);
          }
          tc::mma_commit(&s.mma_bar[st]);
          uses[st] += 1;
        }
        tc::mma_commit(&s.done_bar);
      } else {
        for (int ka = 0; ka < args.katoms; ++ka) uses[ka & 1] += 1;
      }
      tc::mbar_wait(&s.done_bar, dones & 1);
      ++dones;
      tc::fence_after_sync();
      epi_run_chunk(s.ch, nkc, k0, lane_base, sqv, args.guard, run);
      tc::fence_before_sync();
      k0 = k1;
    }
    // ---- routing: one atomic per row (a wide node has up to K children)
    if (my_patch >= 0) {
      if (epi_run_flagged(run)) {
        const int slot = atomicAdd(&args.queue_len[a.depth], 1);
        args.queue[2 * slot] = my_patch;
        args.queue[2 * slot + 1] = u;
      } else {
        level_route(pv, a, s.lv, kids[run.bi], my_patch);
      }
    }
    __syncthreads();  // A is rewritten by the next tile
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace wide

int select_level_wide(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                      cudaStream_t st) {
  FEPLL_REQUIRE(p->have_tc && p->v.P <= 128, "wide tensor level: needs a tcgen05 plan and P <= 128");
  wide::Args args;
  args.a = a;
  args.Z32 = Z32;
  args.z32_pitch = (p->v.P + 31) / 32 * 32;
  args.sq = sq;
  args.guard = guard > 0 ? guard : kDefaultGuard;
  args.queue = p->rs.queue;
  args.queue_len = p->rs.queue_len;
  args.katoms = args.z32_pitch / 32;
  args.nw = args.katoms <= 2 ? 256 : 128;  // A resident + 2 B stages within 227 KB
  const size_t smem = 1024 + 2 * (size_t)args.katoms * wide::kAtomBytes +
                      4 * (size_t)args.nw * 128 + sizeof(wide::Tables);
  FEPLL_CUDA(cudaFuncSetAttribute(wide::select_level_wide_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  wide::select_level_wide_kernel<<<kSMs, wide::kThreads, smem, st>>>(p->v, args);
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll
