// Kernel (b), tensor-core path, warp-specialized pipeline (P <= 64).
//
// Same arithmetic as select_tc.cu (3xTF32 tcgen05 scoring of one tree level,
// certified argmin, FP64 re-scoring of the rest; pkg/src/fepll/tree.py:416-428,
// pkg/src/fepll/gmm.py:323-339), laid out as a persistent pipeline:
//
//   warps 0-7    producers: warp w owns K atom w/4 of the tile's 128 FP32
//                patch rows (kernel (a) output).  Row indices arrive several
//                tiles early by cp.async into a smem ring, rows are prefetched
//                into L2 and then into registers one tile ahead (each load
//                instruction covers four whole 128-byte row atoms); each
//                thread splits TF32 hi/lo and stores 128B-swizzled into one
//                of two A stages.  (A TMA tile::gather4 producer was measured and
//                rejected: ~62 cycles per 512-byte gather4, ~2.3 TB/s chip-wide,
//                tools/tma_rate.cu — below this loop, and it needs the split
//                rows materialized, doubling kernel (a)'s writes.)
//   warp 8       MMA issuer (warp-collective, elected lane): keeps the
//                current node's group image G_u resident in smem (reloaded
//                by the TMA bulk engine only when the node changes — each CTA
//                walks a contiguous, node-sorted tile range), issues 24
//                tcgen05.mma per tile into one of four 128-column TMEM
//                accumulators;
//   warps 9-24   four epilogue groups (tile i -> group i % 4): tcgen05.ld,
//                per-child scores (tc_epi.cuh), certified argmin,
//                aggregated routing.
//
// smem (P=64, N<=128): 2 x 64 KB A stages + 64 KB B + tables; TMEM 512 cols.
#include <algorithm>

#include "route.cuh"
#include "tc.cuh"
#include "tc_epi.cuh"

namespace fepll {

namespace ws {

constexpr int kRows = 128;
constexpr int kProducerWarps = 8;
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;
constexpr int kGroups = 4;                 // epilogue groups == TMEM accumulators
constexpr int kEpiWarps = 4 * kGroups;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kStages = 2;
constexpr int kAtomA = kRows * 128;     // bytes of one K atom of A (hi or lo)
constexpr int kMaxKAtoms = 2;           // P <= 64
constexpr int kMaxN = 128;              // padded group width == accumulator columns
constexpr int kStageBytes = 2 * kMaxKAtoms * kAtomA;       // hi + lo, all atoms
constexpr int kBBytes = 2 * kMaxKAtoms * kMaxN * 128;      // hi + lo, all atoms
constexpr uint32_t kTmemCols = 512;

struct EpiGroup {
  EpiChild ch;
  int node;
  int32_t key[kRows];
  int32_t lrank[kRows];
  int32_t bcnt[kMaxChildren + 1];
  int32_t bbase[kMaxChildren + 1];
};

constexpr int kMaxNodes = 128;  // internal nodes per level handled by this kernel
using WsLevelTables = LevelTablesN<256>;  // next level <= 256 nodes

constexpr int kIdxAhead = 6;   // tiles of row indices in flight per producer thread
constexpr int kIdxRing = 7;
constexpr int kL2Ahead = 3;    // tiles whose rows are prefetched into L2

struct Smem {
  int32_t idx_ring[2][kIdxRing][kRows];  // [K atom group][slot][row]
  WsLevelTables lv;
  int64_t nd_off[kMaxNodes];      // segment offset of each depth-d node (a.off)
  int16_t nd_npad[kMaxNodes];     // padded group width
  int16_t nd_nk[kMaxNodes];       // child count
  EpiGroup epi[kGroups];
  uint64_t a_full[kStages], a_empty[kStages], acc_full[kGroups], acc_empty[kGroups];
  uint64_t b_full, drain;
  uint32_t tmem_base;
  int32_t t_begin, t_end;
};

struct Args {
  LevelArgs a;
  const float* Z32;      // [n_total][z32_pitch] FP32 patch rows (fepll_extract)
  int z32_pitch;
  const double* sq;
  double guard;
  int32_t* queue;
  int32_t* queue_len;
  int katoms;
  uint64_t* trace;       // debug timeline: [CTA][64 tiles][16] clock64 stamps (or NULL)
};

__device__ __forceinline__ void stamp(const Args& a, int i, int slot) {
  if (a.trace && i < 64) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles (per-CTA relative timing)
    a.trace[((size_t)blockIdx.x * 64 + i) * 16 + slot] = t;
  }
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

struct TileInfo {
  int k, u, first, m;
};

// tile -> (level-local node k, BFS id u, first row, rows): smem only
__device__ __forceinline__ TileInfo tile_info(const LevelArgs& a, const WsLevelTables& lv, int tile) {
  TileInfo ti;
  ti.k = prefix_find(lv.tpre, a.lvl_end - a.lvl_begin, tile);
  ti.u = a.lvl_begin + ti.k;
  ti.first = (tile - lv.tpre[ti.k]) * kRows;
  ti.m = min(kRows, (lv.cpre[ti.k + 1] - lv.cpre[ti.k]) - ti.first);
  return ti;
}

// K atom ka of the warp's 32 rows (ring entries rg[0..31]): lane L holds the
// 16-byte chunk L & 7 of rows 4q + L / 8, q = 0..7, so each load instruction
// covers four whole 128-byte row atoms (zeros for g < 0)
__device__ __forceinline__ void load_rows(const Args& args, const int32_t* rg, int ka, int lane,
                                          float4 (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int g = rg[4 * q + (lane >> 3)];
    v[q] = g >= 0 ? __ldg(reinterpret_cast<const float4*>(args.Z32 + (int64_t)g * args.z32_pitch) +
                          ka * 8 + (lane & 7))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
select_level_ws_kernel(PlanView pv, Args args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = tc::align1024(smem_raw);
  uint8_t* stageA = base;
  uint8_t* bbuf = base + kStages * kStageBytes;   // resident B (hi then lo)
  Smem& s = *reinterpret_cast<Smem*>(bbuf + kBBytes);
  const LevelArgs& a = args.a;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (warp == kMmaWarp) tc::tmem_alloc(&s.tmem_base, kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.a_full[i], kProducerWarps);
      tc::mbar_init(&s.a_empty[i], 1);
    }
    for (int i = 0; i < kGroups; ++i) {
      tc::mbar_init(&s.acc_full[i], 1);
      tc::mbar_init(&s.acc_empty[i], 4);
    }
    tc::mbar_init(&s.b_full, 1);
    tc::mbar_init(&s.drain, 1);
    tc::fence_mbar_init();
  }
  if (tid < kGroups) s.epi[tid].node = -1;
  level_tables(pv, a, s.lv, kRows);  // contains __syncthreads
  for (int k = tid; k < a.lvl_end - a.lvl_begin; k += blockDim.x) {
    const int u = a.lvl_begin + k;
    s.nd_off[k] = a.off[u];
    s.nd_npad[k] = (int16_t)pv.tc_npad[u];
    s.nd_nk[k] = (int16_t)pv.child_count[u];
  }
  if (tid == 0) {
    const int T = s.lv.total_tiles;
    s.t_begin = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
    s.t_end = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s.tmem_base;
  const int t_begin = s.t_begin, t_end = s.t_end;
  const int ntile = t_end - t_begin;
  const int t = a.t;

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producers
    const int row = tid & (kRows - 1);
    const int ka = warp >> 2;          // K atom of this warp
    const bool active = ka < args.katoms;
    // Row indices arrive kIdxAhead tiles early by cp.async into a per-thread
    // smem ring (no register dependency), row data one tile ahead in
    // registers.
    int32_t* ring = s.idx_ring[ka][0];
    auto fetch_idx = [&](int j) {  // tile t_begin + j -> ring slot j % kIdxRing
      if (j < ntile) {
        const TileInfo ti = tile_info(a, s.lv, t_begin + j);
        int32_t* dst = ring + (j % kIdxRing) * kRows + row;
        if (row < ti.m) {
          tc::cp_async4(dst, a.seg_in + s.nd_off[ti.k] + ti.first + row);
        } else {
          *dst = -1;
        }
      }
      tc::cp_async_commit();
    };
    float4 v[8];
    if (active) {
      for (int j = 0; j < kIdxAhead; ++j) fetch_idx(j);
      tc::cp_async_wait<0>();
      __syncwarp();  // the other lanes' ring entries
      for (int j = 1; j < kL2Ahead && j < ntile; ++j) {
        const int gp = ring[(j % kIdxRing) * kRows + row];
        if (gp >= 0) tc::prefetch_l2(args.Z32 + (int64_t)gp * args.z32_pitch + ka * 32);
      }
      if (ntile > 0) load_rows(args, ring + 32 * (warp & 3), ka, lane, v);
    }
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      if (i >= kStages) tc::mbar_wait(&s.a_empty[st], ((i / kStages) - 1) & 1);
      if (tid == 0) stamp(args, i, 0);
      if (active) {
        uint8_t* A = stageA + st * kStageBytes + (warp & 3) * 4096;
        const int c = lane & 7;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = 4 * q + (lane >> 3);  // row inside the warp's 32
          const int o = (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
          float4 h, l;
          h.x = tc::to_tf32(v[q].x); l.x = v[q].x - h.x;
          h.y = tc::to_tf32(v[q].y); l.y = v[q].y - h.y;
          h.z = tc::to_tf32(v[q].z); l.z = v[q].z - h.z;
          h.w = tc::to_tf32(v[q].w); l.w = v[q].w - h.w;
          *reinterpret_cast<float4*>(A + (2 * ka) * kAtomA + o) = h;
          *reinterpret_cast<float4*>(A + (2 * ka + 1) * kAtomA + o) = l;
        }
        tc::fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.a_full[st]);
      if (tid == 0) stamp(args, i, 1);
      // prefetch the next tile's row while this one is consumed
      if (active && i + 1 < ntile) {
        fetch_idx(i + kIdxAhead);
        tc::cp_async_wait<kIdxAhead - kL2Ahead>();  // indices through tile i+kL2Ahead landed
        __syncwarp();
        if (i + kL2Ahead < ntile) {
          const int gp = ring[((i + kL2Ahead) % kIdxRing) * kRows + row];
          if (gp >= 0) tc::prefetch_l2(args.Z32 + (int64_t)gp * args.z32_pitch + ka * 32);
        }
        load_rows(args, ring + ((i + 1) % kIdxRing) * kRows + 32 * (warp & 3), ka, lane, v);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs this loop (uniform values); one elected lane
    // issues each tcgen05 instruction (tc.cuh *_warp).
    int cur = -1;
    uint32_t b_loads = 0, drains = 0;
    const uint64_t a_base = tc::desc_sw128(tc::smem_u32(stageA));
    const uint64_t b_base = tc::desc_sw128(tc::smem_u32(bbuf));
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      const int ac = i % kGroups;
      const TileInfo ti = tile_info(a, s.lv, t_begin + i);
      const int npad = s.nd_npad[ti.k];
      const uint32_t bhalf = (uint32_t)args.katoms * npad * 128u;
      if (ti.u != cur) {
        if (i > 0) {  // every MMA reading the old B must be done
          tc::mma_commit_warp(&s.drain);
          tc::mbar_wait(&s.drain, drains & 1);
          ++drains;
        }
        if (lane == 0) {
          tc::mbar_arrive_expect_tx(&s.b_full, 2 * bhalf);
          const int64_t boff = (int64_t)t * pv.tc_tstride + pv.tc_off[ti.u];
          tc::bulk_g2s(bbuf, pv.tc_hi + boff, bhalf, &s.b_full);
          tc::bulk_g2s(bbuf + bhalf, pv.tc_lo + boff, bhalf, &s.b_full);
        }
        __syncwarp();
        tc::mbar_wait(&s.b_full, b_loads & 1);
        ++b_loads;
        cur = ti.u;
      }
      if (i >= kGroups) tc::mbar_wait(&s.acc_empty[ac], ((i / kGroups) - 1) & 1);

      tc::mbar_wait(&s.a_full[st], (i / kStages) & 1);
      tc::fence_after_sync();
      if (lane == 0) stamp(args, i, 2);
      const uint32_t idesc = tc::idesc_tf32(kRows, npad);
      const uint32_t d = tmem + ac * kMaxN;
      // descriptor start-address field counts 16-byte units
      const uint64_t A0 = a_base + (uint64_t)((st * kStageBytes) >> 4);
      for (int kq = 0; kq < args.katoms; ++kq) {
        const uint64_t a_hi = A0 + (uint64_t)(((2 * kq) * kAtomA) >> 4);
        const uint64_t a_lo = A0 + (uint64_t)(((2 * kq + 1) * kAtomA) >> 4);
        const uint64_t b_hi = b_base + (uint64_t)((kq * npad * 128) >> 4);
        const uint64_t b_lo = b_base + (uint64_t)((bhalf + kq * npad * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ko = 2 * kk;  // 8 tf32 = 32 bytes inside the swizzle atom
          const uint32_t acc = (kq > 0 || kk > 0) ? 1u : 0u;
          tc::mma_tf32_warp(d, a_lo + ko, b_hi + ko, idesc, acc);
          tc::mma_tf32_warp(d, a_hi + ko, b_lo + ko, idesc, 1u);
          tc::mma_tf32_warp(d, a_hi + ko, b_hi + ko, idesc, 1u);
        }
      }
      tc::mma_commit_warp(&s.a_empty[st]);
      tc::mma_commit_warp(&s.acc_full[ac]);
      if (lane == 0) stamp(args, i, 3);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - kEpiWarp0;       // 0..15
    const int grp = ew >> 2;               // tiles with i % 4 == grp
    const int row = 32 * (warp & 3) + lane;
    const uint32_t d_acc = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + grp * kMaxN;
    EpiGroup& E = s.epi[grp];
    const int etid = (ew & 3) * 32 + lane;  // 0..127 inside the group
    const int bar_id = 1 + grp;
    const double guard = args.guard;
    for (int i = grp; i < ntile; i += kGroups) {
      const TileInfo ti = tile_info(a, s.lv, t_begin + i);
      const int u = ti.u;
      const int nk = s.nd_nk[ti.k];
      const bool valid = row < ti.m;
      const int g = valid ? a.seg_in[s.nd_off[ti.k] + ti.first + row] : -1;
      const double sqv = valid ? args.sq[g] : 0.0;
      if (u != E.node) {
        named_bar(bar_id, 128);  // everyone done with the previous tables
        epi_load_node(pv, t, u, E.ch, etid, 128);
        named_bar(bar_id, 128);
        if (etid == 0) E.node = u;
      }
      tc::mbar_wait(&s.acc_full[grp], (i / kGroups) & 1);
      tc::fence_after_sync();
      if (etid == 0) stamp(args, i, 4);
      bool flagged;
      const int bi = epi_score_row(E.ch, nk, d_acc, sqv, guard, &flagged);
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.acc_empty[grp]);
      if (etid == 0) stamp(args, i, 5);
      // routing, aggregated over the group's 128 rows
      if (etid <= kMaxChildren) E.bcnt[etid] = 0;
      named_bar(bar_id, 128);
      if (valid) {
        const int key = flagged ? kMaxChildren : bi;
        E.key[row] = key;
        E.lrank[row] = atomicAdd(&E.bcnt[key], 1);
      }
      named_bar(bar_id, 128);
      if (etid < nk && E.bcnt[etid] > 0) E.bbase[etid] = atomicAdd(&a.cnt[E.ch.bfs[etid]], E.bcnt[etid]);
      if (etid == 127 && E.bcnt[kMaxChildren] > 0)
        E.bbase[kMaxChildren] = atomicAdd(&args.queue_len[a.depth], E.bcnt[kMaxChildren]);
      named_bar(bar_id, 128);
      if (valid) {
        const int key = E.key[row];
        const int slot = E.bbase[key] + E.lrank[row];
        if (key == kMaxChildren) {
          args.queue[2 * slot] = g;
          args.queue[2 * slot + 1] = u;
        } else {
          const int v = E.ch.bfs[key];
          const int64_t b0 = s.lv.child_off[v - a.nxt_begin];
          if (pv.child_count[v] > 0) {
            a.seg_out[b0 + slot] = g;
          } else {
            a.leafseg[b0 + slot] = g;
            a.labels[g] = pv.leaf_index[v];
          }
        }
      }
      if (etid == 0) stamp(args, i, 6);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace ws

uint64_t* g_ws_trace = nullptr;
int g_ws_trace_level = -1;

bool select_ws_supported(const Plan* p, int d) {
  const int width = p->level_start[d + 1] - p->level_start[d];
  const int width_next = p->level_start[d + 2] - p->level_start[d + 1];
  return p->have_tc && p->v.P <= 64 && !p->level_wide[d] && p->level_tc_npad[d] <= ws::kMaxN &&
         width <= ws::kMaxNodes && width_next <= ws::WsLevelTables::kCap;
}

// 2-D tensor map over the [rows][pitch] FP32 patch rows: boxes of one
// 128-byte K atom of one row, 128B swizzle (the UMMA K-major layout)
int select_level_ws(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                    cudaStream_t st) {
  ws::Args args;
  args.a = a;
  args.Z32 = Z32;
  args.z32_pitch = (p->v.P + 31) / 32 * 32;
  args.sq = sq;
  args.guard = guard > 0 ? guard : kDefaultGuard;
  args.queue = p->rs.queue;
  args.queue_len = p->rs.queue_len;
  args.katoms = (p->v.P + 31) / 32;
  args.trace = (a.depth == g_ws_trace_level) ? g_ws_trace : nullptr;
  const size_t smem = 1024 + ws::kStages * ws::kStageBytes + ws::kBBytes + sizeof(ws::Smem);
  FEPLL_CUDA(cudaFuncSetAttribute(ws::select_level_ws_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ws::select_level_ws_kernel<<<kSMs, ws::kThreads, smem, st>>>(p->v, args);
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll

extern "C" int fepll_debug_ws_trace(void* device_buffer, int32_t level) {
  fepll::g_ws_trace = static_cast<uint64_t*>(device_buffer);
  fepll::g_ws_trace_level = level;
  return 0;
}
