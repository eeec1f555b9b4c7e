// Kernel (b), tensor-core path, deep-staging variant of select_ws.cu (P <= 64).
//
// Same arithmetic and routing as select_ws.cu (3xTF32 tcgen05 scoring of one
// tree level, certified argmin, FP64 re-scoring of the rest;
// pkg/src/fepll/tree.py:416-428, pkg/src/fepll/gmm.py:323-339); the operand
// staging differs:
//
//   * tcgen05 kind::tf32 reads only the top 19 bits of an FP32 operand
//     (truncation, tools/tf32_trunc_test.cu), so the raw FP32 patch row is
//     the hi operand as is.  Four loader warps pull the rows by cp.async
//     (every instruction moves four whole 128-byte row atoms) into one of
//     four 32 KB raw stages and signal the stage's mbarrier when the copies
//     land (cp.async.mbarrier.arrive) — three tiles of loads in flight, no
//     register staging, no loader waiting on anything but a free stage;
//   * the score is z . b = z_hi . b_hi + (z_hi . b_lo + z_lo . b_hi) with
//     z_hi = trunc_tf32(z) (what kind::tf32 reads from the raw stage), b_hi
//     = rne_tf32(b): the main term is one kind::tf32 pass (A = raw stage),
//     the two small cross terms one kind::f16 pass in bf16 with K doubled —
//     A' = [bf16(z_hi) | bf16(z_lo)] against B' = [bf16(b_lo) | bf16(b_hi)]
//     (plan.py bf16_cross_image).  A bf16 MMA of K = 16 costs what a tf32
//     MMA of K = 8 does, so the pair costs 2 tf32 passes instead of 3xTF32's
//     three, and the cross pass reads only B from shared memory;
//   * eight converter warps build A' (per thread: one 128-byte K atom of one
//     row) and write it to tensor memory with tcgen05.st (two 64-column
//     buffers);
//   * NG accumulators of ACC columns / epilogue groups (512 TMEM columns in
//     all with the A' buffers).
//
// Error budget (per element, |z_lo| < 2^-10 |z|, |b_lo| <= 2^-11 |b|, bf16
// rounding <= 2^-9 relative): z_hi b_lo in bf16 <= 2^-19 |z||b|, z_lo b_hi
// in bf16 <= 2^-18 |z||b|, the dropped z_lo b_lo <= 2^-21 |z||b|, FP32
// accumulation over 16 MMAs <= 2^-19: in all < 2^-17 ||z|| ||b|| by
// Cauchy-Schwarz — twice the 3xTF32 projection bound of tc_epi.cuh, so this
// kernel certifies with twice the guard (2^-15 by default).
#include <algorithm>

#include "route.cuh"
#include "tc.cuh"
#include "tc_epi.cuh"

namespace fepll {

namespace ws2 {
constexpr int kRows = 128;
// warp roles for LW loader warps: warps 0..LW-1 load (warp w: rows
// 128/LW * w .., both K atoms), the next 8 convert (K atom, TMEM lane quarter
// w % 4), then the MMA issuer, then 4 NG epilogue warps.  Four loader warps
// issue a tile's 2048 cp.async 10-15 % faster than two (levels 320 -> 288 us
// at 64 x 1024^2); eight measured no faster (the LSU, not the issuing warps,
// is then the limit: tools/ldgsts_rate.cu, 0.98 vs 0.90 us per tile alone)
template <int LW>
struct Roles {
  static constexpr int kLoaderWarps = LW;
  static constexpr int kLoaderRows = kRows / LW;
  static constexpr int kLoaderQ = kLoaderRows / 4;  // rows per lane (4 rows per instruction)
  static constexpr int kLoaderThreads = 32 * LW;
  static constexpr int kConvWarp0 = LW;
  static constexpr int kConvWarps = 8;
  static constexpr int kMmaWarp = kConvWarp0 + kConvWarps;
  static constexpr int kEpiWarp0 = kMmaWarp + 1;
};
// + (SCHED) one scheduler warp after the epilogue warps: it walks the tiles
// ahead of the MMA issuer, waits on every tile's barriers (raw stage landed,
// lo written, accumulator free) and publishes the tile's node and width with
// one mbarrier, so the issuer's loop between two tiles' MMAs is one wait.
// Measured: levels on the four-group <4, 96> kernel 286 -> 268 us and
// 348 -> 322 us; the three-group <3, 128> kernel, whose epilogue groups are
// the limit, got slower (292 -> 310 us), so it keeps the issuer-side waits.
// epilogue groups (== TMEM accumulators) and accumulator width are template
// parameters: <3, 128> for levels with nodes up to 128 padded columns,
// <4, 96> where every node fits 96 (four groups keep up with the MMAs)
constexpr int threads_for(int ng, int lw, bool sched) {
  return (Roles<1>::kEpiWarp0 - 1 + lw + 4 * ng + (sched ? 1 : 0)) * 32;
}
constexpr int kReady = 4;  // scheduler -> issuer ring
constexpr int kStages = 4;              // raw row stages (hi operand)
constexpr int kLoBufs = 2;              // TMEM lo buffers
constexpr int kAtomA = kRows * 128;     // bytes of one K atom of A
constexpr int kMaxKAtoms = 2;           // P <= 64
constexpr int kMaxN = 128;              // padded group width == accumulator columns
constexpr int kStageBytes = kMaxKAtoms * kAtomA;           // raw rows, all atoms
constexpr int kBBytes = 2 * kMaxKAtoms * kMaxN * 128;      // hi + lo, all atoms
constexpr uint32_t kTmemCols = 512;

// Routing is deferred by one group iteration: tile j's segment bases come
// back from the contended global atomics while tile j+kGroups is scored, and
// tile j's indices are written then.  Counts / bases are triple-buffered by
// the group's iteration so one named barrier per tile suffices.
struct EpiGroup {
  EpiChild ch;
  int node;
  int32_t bcnt[3][kMaxChildren + 1];
  int32_t bbase[3][kMaxChildren + 1];
};

constexpr int kMaxNodes = 128;  // internal nodes per level handled by this kernel
using WsLevelTables = LevelTablesN<256>;  // next level <= 256 nodes

constexpr int kPrefetch = 3;   // tiles ahead of its cp.async a row is prefetched into L2
// tiles of row indices in flight ahead of their rows: the prefetch of tile
// i + kPrefetch waits for its indices without waiting for recent row copies
constexpr int kIdxAhead = 6 + kPrefetch;
constexpr int kIdxRing = kIdxAhead + 1;

template <int NG>
struct Smem {
  int32_t idx_ring[kIdxRing][kRows];     // [slot][row]
  WsLevelTables lv;
  int64_t nd_off[kMaxNodes];      // segment offset of each depth-d node (a.off)
  int16_t nd_npad[kMaxNodes];     // padded group width
  int16_t nd_nk[kMaxNodes];       // child count
  EpiGroup epi[NG];
  // mma_done[i % kStages]: tile i's MMAs finished — frees its raw stage and
  // its lo buffer (kLoBufs divides kStages)
  uint64_t raw_full[kStages], mma_done[kStages], lo_full[kLoBufs];
  uint64_t acc_full[NG], acc_empty[NG];
  uint64_t b_full, drain;
  uint64_t ready[kReady];       // scheduler: tile i's barriers passed, tinfo[i % kReady] valid
  int32_t tinfo_u[kReady], tinfo_npad[kReady];
  uint32_t tmem_base;
  int32_t t_begin, t_end;
};

static_assert(1024 + kStages * kStageBytes + kBBytes + sizeof(Smem<4>) <= 232448 &&
                  1024 + kStages * kStageBytes + kBBytes + sizeof(Smem<3>) <= 232448,
              "ws2 shared memory exceeds 227 KB");

struct Args {
  LevelArgs a;
  const float* Z32;      // [n_total][z32_pitch] FP32 patch rows (fepll_extract)
  int z32_pitch;
  const double* sq;
  double guard;
  int32_t* queue;
  int32_t* queue_len;
  // deferred verification (vq != NULL): uncertified rows are routed by
  // their tensor-core argmin like the certified ones and logged to vq
  int4* vq;
  int32_t* vq_len;
  int64_t vq_cap;
  int32_t* pos_leaf;
  int perturb;           // test hook (plan option defer_test): uncertified rows take the next child
  int katoms;
  int prefetch;          // tiles ahead whose rows the loaders prefetch into L2 (0: off)
  uint64_t* trace;       // debug timeline: [CTA][64 tiles][16] clock64 stamps (or NULL)
  uint64_t* spans;       // debug: [CTA][4] globaltimer at entry, after the prologue, at the end (or NULL)
};

__device__ __forceinline__ void stamp(const Args& a, int i, int slot) {
  if (a.trace && i < 64) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles (per-CTA relative timing)
    a.trace[((size_t)blockIdx.x * 64 + i) * 16 + slot] = t;
  }
}

__device__ __forceinline__ void span_stamp(const Args& a, int slot) {
  if (a.spans && threadIdx.x == 0) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.spans[(size_t)blockIdx.x * 4 + slot] = g;
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

// tile -> (level-local node k, BFS id u, first row, rows): smem only.  Every
// role walks its tiles in increasing order, so the node index advances
// instead of being searched for (the MMA warp's per-tile bookkeeping sits
// between its MMA batches, where the tensor pipe would idle).
struct TileCursor {
  int k = -1;
  __device__ __forceinline__ TileInfo at(const LevelArgs& a, const WsLevelTables& lv, int tile) {
    const int n = a.lvl_end - a.lvl_begin;
    if (k < 0) k = prefix_find(lv.tpre, n, tile);
    while (k + 1 < n && lv.tpre[k + 1] <= tile) ++k;
    TileInfo ti;
    ti.k = k;
    ti.u = a.lvl_begin + k;
    ti.first = (tile - lv.tpre[k]) * kRows;
    ti.m = min(kRows, (lv.cpre[k + 1] - lv.cpre[k]) - ti.first);
    return ti;
  }
};

template <int NG, int ACC, int LW, bool SCHED>
__global__ void __launch_bounds__(threads_for(NG, LW, SCHED), 1)
select_level_ws2_kernel(PlanView pv, Args args) {
  using R = Roles<LW>;
  constexpr int kLoaderWarps = R::kLoaderWarps, kLoaderRows = R::kLoaderRows, kLoaderQ = R::kLoaderQ;
  constexpr int kLoaderThreads = R::kLoaderThreads, kConvWarp0 = R::kConvWarp0;
  constexpr int kConvWarps = R::kConvWarps, kMmaWarp = R::kMmaWarp, kEpiWarp0 = R::kEpiWarp0;
  constexpr int kGroups = NG;
  constexpr int kAcc = ACC;                          // accumulator columns (>= node width)
  constexpr uint32_t kXCol0 = NG * ACC;              // TMEM column of A' buffer 0
  static_assert(NG * ACC + kLoBufs * 64 <= 512, "TMEM: accumulators + A' buffers");
  static_assert(kStages % kLoBufs == 0, "mma_done serves both rings");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = tc::align1024(smem_raw);
  uint8_t* stageA = base;
  uint8_t* bbuf = base + kStages * kStageBytes;   // resident B (hi then lo)
  Smem<NG>& s = *reinterpret_cast<Smem<NG>*>(bbuf + kBBytes);
  const LevelArgs& a = args.a;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  span_stamp(args, 0);

  if (warp == kMmaWarp) tc::tmem_alloc(&s.tmem_base, kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.raw_full[i], kLoaderThreads);
      tc::mbar_init(&s.mma_done[i], 1);
    }
    for (int i = 0; i < kLoBufs; ++i) {
      tc::mbar_init(&s.lo_full[i], kConvWarps);
    }
    for (int i = 0; i < kGroups; ++i) {
      tc::mbar_init(&s.acc_full[i], 1);
      tc::mbar_init(&s.acc_empty[i], 4);
    }
    tc::mbar_init(&s.b_full, 1);
    for (int i = 0; i < kReady; ++i) tc::mbar_init(&s.ready[i], 1);
    tc::mbar_init(&s.drain, 1);
    tc::fence_mbar_init();
  }
  if (tid < kGroups) s.epi[tid].node = -1;
  // launched with PDL behind the previous level's re-scoring: everything
  // above (TMEM, barriers) overlapped its tail; the counts are its output
  pdl_wait();
  pdl_trigger();  // the re-scoring grid may queue behind this one's CTAs
  level_tables_warp(pv, a, s.lv, kRows);  // ends with a __syncthreads (nodes <= 256 on both sides)
  if (warp == 0) {
    // node tables (four nodes per lane) and, from them, contiguous tile
    // ranges of equal estimated cost: a tile costs 16 + npad / 8 (loads,
    // epilogue and MMAs of its node's width) — on the leaf level of the cfg5
    // tree the 4-child nodes' tiles (128 columns) take ~15 % longer than the
    // 3-child ones (96), and equal tile counts left the CTAs holding them
    // 40 us behind.  One warp with a shuffle scan: one thread walking the
    // nodes twice cost ~5 us of every CTA's prologue at 8 nodes and ~10 us
    // at 64, and filling the tables from every thread one more CTA barrier.
    static_assert(kMaxNodes <= 128, "four nodes per lane");
    const int nd = a.lvl_end - a.lvl_begin;
    const int T = s.lv.total_tiles;
    int npad_r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * lane + q;
      npad_r[q] = 0;
      if (k < nd) {
        const int u = a.lvl_begin + k;
        npad_r[q] = pv.tc_npad[u];
        s.nd_off[k] = a.off[u];
        s.nd_npad[k] = (int16_t)npad_r[q];
        s.nd_nk[k] = (int16_t)pv.child_count[u];
      }
    }
    const int npad0 = __shfl_sync(0xffffffffu, npad_r[0], 0);
    int64_t c[4];
    int wk[4];
    int64_t sum = 0;
    bool mix = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * lane + q;
      c[q] = 0;
      wk[q] = 1;
      if (k < nd) {
        wk[q] = 16 + npad_r[q] / 8;
        c[q] = (int64_t)(s.lv.tpre[k + 1] - s.lv.tpre[k]) * wk[q];
        mix |= npad_r[q] != npad0;
      }
      sum += c[q];
    }
    int64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t W = __shfl_sync(0xffffffffu, incl, 31);
    const bool mixed = __any_sync(0xffffffffu, mix);
    if (!mixed) {
      if (lane == 0) {
        s.t_begin = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
        s.t_end = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);
      }
    } else {
      const int64_t x0 = W * blockIdx.x / gridDim.x, x1 = W * (blockIdx.x + 1) / gridDim.x;
      int64_t acc = incl - sum;
      int tb = T, te = T;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 4 * lane + q;
        const int64_t nxt = acc + c[q];
        // the first node whose cost range holds x: acc <= x < nxt (empty nodes have nxt == acc)
        if (acc <= x0 && x0 < nxt) tb = s.lv.tpre[k] + (int)((x0 - acc + wk[q] - 1) / wk[q]);
        if (acc <= x1 && x1 < nxt) te = s.lv.tpre[k] + (int)((x1 - acc + wk[q] - 1) / wk[q]);
        acc = nxt;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tb = min(tb, __shfl_xor_sync(0xffffffffu, tb, o));
        te = min(te, __shfl_xor_sync(0xffffffffu, te, o));
      }
      if (lane == 0) {
        s.t_begin = min(tb, T);
        s.t_end = blockIdx.x + 1 == gridDim.x ? T : min(te, T);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s.tmem_base;
  const int t_begin = s.t_begin, t_end = s.t_end;
  span_stamp(args, 1);
  if (args.trace && tid == 0) {  // CTA span on the global clock (load-balance check)
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    args.trace[((size_t)blockIdx.x * 64 + 63) * 16 + 14] = g;
  }
  const int ntile = t_end - t_begin;
  const int t = a.t;

  if (warp < kLoaderWarps) {
    // ------------------------------------------------------------ loaders
    // Row indices arrive kIdxAhead tiles early (cp.async into the ring, one
    // commit group per tile); each lane then issues 32 cp.async of 16 bytes
    // (the warp's 64 rows x 2 K atoms, four whole row atoms per instruction)
    // and arrives on raw_full once they land.
    const int r0 = kLoaderRows * warp;
    TileCursor cur_idx;
    auto issue_idx = [&](int j) {
      if (j < ntile) {
        const TileInfo ti = cur_idx.at(a, s.lv, t_begin + j);
        int32_t* ring = s.idx_ring[j % kIdxRing];
#pragma unroll
        for (int h = 0; h < (kLoaderRows + 31) / 32; ++h) {
          if (32 * h + lane >= kLoaderRows) break;
          const int row = r0 + 32 * h + lane;
          if (row < ti.m) tc::cp_async4(ring + row, a.seg_in + s.nd_off[ti.k] + ti.first + row);
          else ring[row] = -1;
        }
      }
    };
    const int c16 = lane & 7;
    const int64_t pitch = args.z32_pitch;
    for (int j = 0; j < kIdxAhead; ++j) {
      issue_idx(j);
      tc::cp_async_commit();
    }
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      if (i >= kStages) tc::mbar_wait(&s.mma_done[st], ((i / kStages) - 1) & 1);
      if (tid == 0) stamp(args, i, 8);
      if (args.prefetch > 0) {
        // idx(i + kPrefetch) landed (and with it idx(i)); each lane sends its
        // row of that tile to L2 now, so the stage's cp.async later hits L2:
        // DRAM requests stay in flight beyond the smem stages' capacity
        tc::cp_async_wait<kIdxAhead - 1 - kPrefetch>();
        const int jp = i + kPrefetch;
        if (jp < ntile) {
          const int gp = s.idx_ring[jp % kIdxRing][r0 + lane];
          if (lane < kLoaderRows && gp >= 0) {
            const float* rowp = args.Z32 + (int64_t)gp * pitch;
            if (args.prefetch == 2) {
              tc::prefetch_l2_bulk(rowp, (uint32_t)(args.katoms * 128));
            } else {
              for (int ka = 0; ka < args.katoms; ++ka) tc::prefetch_l2(rowp + 32 * ka);
            }
          }
        }
      } else {
        tc::cp_async_wait<kIdxAhead - 1>();  // idx(i) landed (one group per tile)
      }
      __syncwarp();                         // ... including the other lanes' entries
      const int32_t* rg = s.idx_ring[i % kIdxRing] + r0;
      int g[kLoaderQ];
#pragma unroll
      for (int q = 0; q < kLoaderQ; ++q) g[q] = rg[4 * q + (lane >> 3)];
      uint8_t* stg = stageA + st * kStageBytes + (r0 >> 3) * 1024;
#pragma unroll
      for (int ka = 0; ka < kMaxKAtoms; ++ka) {
        if (ka < args.katoms) {
          const float* zb = args.Z32 + ka * 32 + 4 * c16;
#pragma unroll
          for (int q = 0; q < kLoaderQ; ++q) {
            const int r = 4 * q + (lane >> 3);  // row inside the warp's rows
            uint8_t* dst = stg + ka * kAtomA + (r >> 3) * 1024 + (r & 7) * 128 + ((c16 ^ (r & 7)) << 4);
            // rows past the tile's end land as zeros (no bytes read)
            tc::cp_async16_zfill(dst, g[q] >= 0 ? zb + g[q] * pitch : args.Z32, g[q] >= 0 ? 16u : 0u);
          }
        }
      }
      issue_idx(i + kIdxAhead);
      tc::cp_async_commit();
      tc::cp_async_mbar_arrive(&s.raw_full[st]);
      if (tid == 0) stamp(args, i, 7);
    }
    tc::cp_async_wait<0>();
  } else if (warp < kConvWarp0 + kConvWarps) {
    // ------------------------------------------------------------ converters
    // thread = one 128-byte K atom of one row; TMEM lane quarter = warp % 4
    const int cw = warp - kConvWarp0;
    const int ka = cw >> 2;
    const int quarter = warp & 3;
    const int row = 32 * quarter + lane;
    const bool active = ka < args.katoms;
    const int r8 = row & 7;
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages, lb = i % kLoBufs;
      tc::mbar_wait(&s.raw_full[st], (i / kStages) & 1);
      if (cw == 0 && lane == 0) stamp(args, i, 0);
      if (i >= kLoBufs) {  // tile i - kLoBufs's MMAs have read lo buffer lb
        const int j = i - kLoBufs;
        tc::mbar_wait(&s.mma_done[j % kStages], (j / kStages) & 1);
      }
      tc::fence_after_sync();
      if (active) {
        const uint8_t* src = stageA + st * kStageBytes + ka * kAtomA + (row >> 3) * 1024 + r8 * 128;
        uint32_t xh[16], xl[16];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = *reinterpret_cast<const float4*>(src + ((c ^ r8) << 4));
          const float h0 = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
          const float h1 = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
          const float h2 = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
          const float h3 = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
          xh[2 * c] = tc::pack_bf16x2(h0, h1);
          xh[2 * c + 1] = tc::pack_bf16x2(h2, h3);
          xl[2 * c] = tc::pack_bf16x2(x.x - h0, x.y - h1);  // exact differences
          xl[2 * c + 1] = tc::pack_bf16x2(x.z - h2, x.w - h3);
        }
        // A' columns: bf16(z_hi) pairs of atom ka at 16 ka, bf16(z_lo) at
        // 16 (katoms + ka)
        const uint32_t xb = tmem + lane_off + kXCol0 + lb * 64;
        tc::tmem_st16(xb + 16 * ka, xh);
        tc::tmem_st16(xb + 16 * (args.katoms + ka), xl);
        tc::tmem_st_wait();
      }
      tc::fence_proxy_async_smem();  // the landed raw stage, for the MMAs' async-proxy reads
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.lo_full[lb]);
      if (cw == 0 && lane == 0) stamp(args, i, 1);
    }
  } else if (!SCHED && warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs this loop (uniform values); one elected lane
    // issues each tcgen05 instruction (tc.cuh *_warp).
    int cur = -1;
    uint32_t b_loads = 0, drains = 0;
    TileCursor tcur;
    const uint64_t a_base = tc::desc_sw128(tc::smem_u32(stageA));
    const uint64_t b_base = tc::desc_sw128(tc::smem_u32(bbuf));
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      const int ac = i % kGroups;
      const TileInfo ti = tcur.at(a, s.lv, t_begin + i);
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
          tc::bulk_g2s(bbuf + bhalf, pv.tc_x + boff, bhalf, &s.b_full);
        }
        __syncwarp();
        tc::mbar_wait(&s.b_full, b_loads & 1);
        ++b_loads;
        cur = ti.u;
      }
      if (lane == 0) stamp(args, i, 10);
      if (i >= kGroups) tc::mbar_wait(&s.acc_empty[ac], ((i / kGroups) - 1) & 1);
      if (lane == 0) stamp(args, i, 9);
      const uint32_t d = tmem + ac * kAcc;
      // main term: z_hi . b_hi, A = the raw stage (cp.async writes: proxy
      // fence after observing them land)
      tc::mbar_wait(&s.raw_full[st], (i / kStages) & 1);
      tc::fence_after_sync();
      tc::fence_proxy_async_smem();
      if (lane == 0) stamp(args, i, 2);
      const uint32_t idesc = tc::idesc_tf32(kRows, npad);
      // descriptor start-address field counts 16-byte units
      const uint64_t A0 = a_base + (uint64_t)((st * kStageBytes) >> 4);
      for (int kq = 0; kq < args.katoms; ++kq) {
        const uint64_t a_hi = A0 + (uint64_t)((kq * kAtomA) >> 4);
        const uint64_t b_hi = b_base + (uint64_t)((kq * npad * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ko = 2 * kk;  // 8 tf32 = 32 bytes inside the swizzle atom
          tc::mma_tf32_warp(d, a_hi + ko, b_hi + ko, idesc, (kq > 0 || kk > 0) ? 1u : 0u);
        }
      }
      // cross terms: A' (TMEM, bf16 pairs) . B' (bf16, K = 2 Ppad)
      const int lb = i % kLoBufs;
      tc::mbar_wait(&s.lo_full[lb], (i / kLoBufs) & 1);
      tc::fence_after_sync();
      const uint32_t idesc16 = tc::idesc_bf16(kRows, npad);
      const uint32_t a_x = tmem + kXCol0 + lb * 64;
      const uint64_t b_x = b_base + (uint64_t)(bhalf >> 4);
      for (int kq = 0; kq < args.katoms; ++kq) {  // B' atom kq: 64 bf16 of K
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)             // K = 16 = 32 bytes per MMA
          tc::mma_bf16_tmemA_warp(d, a_x + 32 * kq + 8 * kk,
                                  b_x + (uint64_t)((kq * npad * 128 + 32 * kk) >> 4), idesc16, 1u);
      }
      tc::mma_commit_warp(&s.mma_done[st]);
      tc::mma_commit_warp(&s.acc_full[ac]);
      if (lane == 0) stamp(args, i, 3);
    }
  } else if (SCHED && warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs this loop (uniform values); one elected lane
    // issues each tcgen05 instruction (tc.cuh *_warp).  Per tile: one wait
    // (the scheduler's ready), the node's B image when it changes, 16 MMAs.
    int cur = -1;
    uint32_t b_loads = 0, drains = 0;
    const uint64_t a_base = tc::desc_sw128(tc::smem_u32(stageA));
    const uint64_t b_base = tc::desc_sw128(tc::smem_u32(bbuf));
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      const int ac = i % kGroups;
      tc::mbar_wait(&s.ready[i % kReady], (i / kReady) & 1);
      const int u = s.tinfo_u[i % kReady];
      const int npad = s.tinfo_npad[i % kReady];
      const uint32_t bhalf = (uint32_t)args.katoms * npad * 128u;
      if (u != cur) {
        if (i > 0) {  // every MMA reading the old B must be done
          tc::mma_commit_warp(&s.drain);
          tc::mbar_wait(&s.drain, drains & 1);
          ++drains;
        }
        if (lane == 0) {
          tc::mbar_arrive_expect_tx(&s.b_full, 2 * bhalf);
          const int64_t boff = (int64_t)t * pv.tc_tstride + pv.tc_off[u];
          tc::bulk_g2s(bbuf, pv.tc_hi + boff, bhalf, &s.b_full);
          tc::bulk_g2s(bbuf + bhalf, pv.tc_x + boff, bhalf, &s.b_full);
        }
        __syncwarp();
        tc::mbar_wait(&s.b_full, b_loads & 1);
        ++b_loads;
        cur = u;
      }
      const uint32_t d = tmem + ac * kAcc;
      // raw stage (cp.async writes; the converters fenced the async proxy
      // after observing it land) and lo buffer observed through ready
      tc::fence_after_sync();
      tc::fence_proxy_async_smem();
      if (lane == 0) stamp(args, i, 2);
      const uint32_t idesc = tc::idesc_tf32(kRows, npad);
      // descriptor start-address field counts 16-byte units
      const uint64_t A0 = a_base + (uint64_t)((st * kStageBytes) >> 4);
      for (int kq = 0; kq < args.katoms; ++kq) {
        const uint64_t a_hi = A0 + (uint64_t)((kq * kAtomA) >> 4);
        const uint64_t b_hi = b_base + (uint64_t)((kq * npad * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ko = 2 * kk;  // 8 tf32 = 32 bytes inside the swizzle atom
          tc::mma_tf32_warp(d, a_hi + ko, b_hi + ko, idesc, (kq > 0 || kk > 0) ? 1u : 0u);
        }
      }
      // cross terms: A' (TMEM, bf16 pairs) . B' (bf16, K = 2 Ppad)
      const int lb = i % kLoBufs;
      const uint32_t idesc16 = tc::idesc_bf16(kRows, npad);
      const uint32_t a_x = tmem + kXCol0 + lb * 64;
      const uint64_t b_x = b_base + (uint64_t)(bhalf >> 4);
      for (int kq = 0; kq < args.katoms; ++kq) {  // B' atom kq: 64 bf16 of K
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)             // K = 16 = 32 bytes per MMA
          tc::mma_bf16_tmemA_warp(d, a_x + 32 * kq + 8 * kk,
                                  b_x + (uint64_t)((kq * npad * 128 + 32 * kk) >> 4), idesc16, 1u);
      }
      tc::mma_commit_warp(&s.mma_done[st]);
      tc::mma_commit_warp(&s.acc_full[ac]);
      if (lane == 0) stamp(args, i, 3);
    }
  } else if (SCHED && warp == kEpiWarp0 + 4 * kGroups) {
    // ------------------------------------------------------------ scheduler
    // tile i: its raw stage landed (raw_full), its lo buffer is written
    // (lo_full), its accumulator drained by the epilogue (acc_empty) and its
    // ready slot consumed (the issuer committed tile i - kReady: mma_done);
    // then node + width go to the issuer through ready[i % kReady]
    TileCursor tcur;
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages, ac = i % kGroups, lb = i % kLoBufs;
      const TileInfo ti = tcur.at(a, s.lv, t_begin + i);
      if (i >= kReady) {
        const int j = i - kReady;
        tc::mbar_wait(&s.mma_done[j % kStages], (j / kStages) & 1);
      }
      if (lane == 0) stamp(args, i, 10);
      if (i >= kGroups) tc::mbar_wait(&s.acc_empty[ac], ((i / kGroups) - 1) & 1);
      if (lane == 0) stamp(args, i, 9);
      tc::mbar_wait(&s.raw_full[st], (i / kStages) & 1);
      tc::mbar_wait(&s.lo_full[lb], (i / kLoBufs) & 1);
      if (lane == 0) {
        s.tinfo_u[i % kReady] = ti.u;
        s.tinfo_npad[i % kReady] = s.nd_npad[ti.k];
        mbar_arrive(&s.ready[i % kReady]);  // release: the slot's writes above
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - kEpiWarp0;       // 0 .. 4 NG - 1
    const int grp = ew >> 2;               // tiles with i % kGroups == grp
    const int row = 32 * (warp & 3) + lane;
    const uint32_t d_acc = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + grp * kAcc;
    EpiGroup& E = s.epi[grp];
    const int etid = (ew & 3) * 32 + lane;  // 0..127 inside the group
    const int bar_id = 1 + grp;
    const double guard = args.guard;
    // pending (previous tile's) route of this thread's row
    bool p_valid = false, p_fl = false;
    int p_kind = 0, p_key = 0, p_lrank = 0, p_g = 0, p_u = 0, p_leaf = 0, p_lrank2 = 0, p_v = 0;
    const bool defer = args.vq != nullptr;
    double p_sq = 0.0;
    int64_t p_b0 = 0;
    int res = 0, res_key = -1;  // this thread's in-flight global atomic (count reservation)
    int it = 0;
    for (int k = etid; k < 3 * (kMaxChildren + 1); k += 128) (&E.bcnt[0][0])[k] = 0;
    named_bar(bar_id, 128);
    auto flush = [&](int buf) {  // write the pending row with bases bbase[buf]
      if (!p_valid) return;
      const int slot = E.bbase[buf][p_key] + p_lrank;
      if (p_kind == 0) {
        args.queue[2 * slot] = p_g;
        args.queue[2 * slot + 1] = p_u;
      } else if (p_kind == 1) {
        a.seg_out[p_b0 + slot] = p_g;
        if (a.sq_out) a.sq_out[p_b0 + slot] = p_sq;
      } else {
        a.leafseg[p_b0 + slot] = p_g;
        a.labels[p_g] = p_leaf;
        if (defer) args.pos_leaf[p_g] = (int32_t)(p_b0 + slot);
      }
      if (p_fl) {  // deferred: the provisional decision, verified after the last level
        const int64_t s2 = (int64_t)E.bbase[buf][kMaxChildren] + p_lrank2;
        if (s2 < args.vq_cap) args.vq[s2] = make_int4(p_g, p_u, a.depth, p_v);
        else atomicOr(&args.queue_len[kMaxDepth - 1], 1);  // overflow (host raises)
      }
    };
    TileCursor tcur;
    for (int i = grp; i < ntile; i += kGroups, ++it) {
      const int cb = it % 3, pb = (it + 2) % 3, nb = (it + 1) % 3;
      const TileInfo ti = tcur.at(a, s.lv, t_begin + i);
      const int u = ti.u;
      const int nk = s.nd_nk[ti.k];
      const bool valid = row < ti.m;
      const int64_t spos = s.nd_off[ti.k] + ti.first + row;  // segment position
      const int g = valid ? a.seg_in[spos] : -1;
      const double sqv = valid ? (a.sq_in ? a.sq_in[spos] : args.sq[g]) : 0.0;
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
      int bi = epi_score_row(E.ch, nk, d_acc, sqv, guard, &flagged);
      // test hook: route the uncertified rows provisionally to a wrong child,
      // so the verification must repair every one of them
      if (defer && args.perturb && flagged && nk > 1) bi = bi + 1 < nk ? bi + 1 : 0;
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.acc_empty[grp]);
      if (etid == 0) stamp(args, i, 5);
      // previous tile's reservations land in bbase[pb]; next buffer zeroed
      if (res_key >= 0) E.bbase[pb][res_key] = res;
      if (etid <= kMaxChildren) E.bcnt[nb][etid] = 0;
      // warp-aggregated local ranks of this tile's rows per key
      const int key = valid ? ((flagged && !defer) ? kMaxChildren : bi) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(peers) - 1;
      int wbase = 0;
      if (key >= 0 && lane == leader) wbase = atomicAdd(&E.bcnt[cb][key], __popc(peers));
      wbase = __shfl_sync(0xffffffffu, wbase, leader);
      const int lrank = wbase + __popc(peers & ((1u << lane) - 1u));
      // deferred: the uncertified rows also take a verify-log slot
      int lrank2 = 0;
      if (defer) {
        const unsigned fl = __ballot_sync(0xffffffffu, valid && flagged);
        if (fl) {
          const int fl_lead = __ffs(fl) - 1;
          int b2 = 0;
          if (lane == fl_lead) b2 = atomicAdd(&E.bcnt[cb][kMaxChildren], __popc(fl));
          b2 = __shfl_sync(0xffffffffu, b2, fl_lead);
          lrank2 = b2 + __popc(fl & ((1u << lane) - 1u));
        }
      }
      named_bar(bar_id, 128);  // counts of this tile complete, bases of the previous visible
      // reserve this tile's segment ranges (results used next iteration)
      res_key = -1;
      if (etid < nk && E.bcnt[cb][etid] > 0) {
        res = atomicAdd(&a.cnt[E.ch.bfs[etid]], E.bcnt[cb][etid]);
        res_key = etid;
      } else if (etid == 127 && E.bcnt[cb][kMaxChildren] > 0) {
        if (defer) {
          res = atomicAdd(args.vq_len, E.bcnt[cb][kMaxChildren]);
          atomicAdd(&args.queue_len[a.depth], E.bcnt[cb][kMaxChildren]);  // per-level statistics
        } else {
          res = atomicAdd(&args.queue_len[a.depth], E.bcnt[cb][kMaxChildren]);
        }
        res_key = kMaxChildren;
      }
      // write the previous tile's rows
      flush(pb);
      // this tile's row becomes pending
      p_valid = valid;
      p_fl = defer && valid && flagged;
      if (valid) {
        p_key = key;
        p_lrank = lrank;
        p_lrank2 = lrank2;
        p_g = g;
        p_sq = sqv;
        p_u = u;
        if (key == kMaxChildren) {
          p_kind = 0;
        } else {
          const int v = E.ch.bfs[key];
          p_v = v;
          p_b0 = s.lv.child_off[v - a.nxt_begin];
          p_kind = pv.child_count[v] > 0 ? 1 : 2;
          p_leaf = pv.leaf_index[v];
        }
      }
      if (etid == 0) stamp(args, i, 6);
    }
    // drain: the last tile's reservations, then its rows
    if (res_key >= 0) E.bbase[(it + 2) % 3][res_key] = res;
    named_bar(bar_id, 128);
    flush((it + 2) % 3);
  }
  tc::fence_before_sync();
  __syncthreads();
  span_stamp(args, 2);
  if (args.trace && tid == 0) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    args.trace[((size_t)blockIdx.x * 64 + 63) * 16 + 15] = g;
  }
  if (warp == kMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace ws2


extern uint64_t* g_ws_trace;
extern int g_ws_trace_level;
bool deferred_verify(const Plan* p);
uint64_t* g_level_spans = nullptr;  // fepll_debug_level_spans: [depth][CTA][4]

int select_level_ws2(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                     cudaStream_t st) {
  ws2::Args args;
  args.a = a;
  args.Z32 = Z32;
  args.z32_pitch = (p->v.P + 31) / 32 * 32;
  args.sq = sq;
  // the mixed-precision projection error is twice 3xTF32's (header)
  args.guard = 2.0 * (guard > 0 ? guard : kDefaultGuard);
  args.queue = p->rs.queue;
  args.queue_len = p->rs.queue_len;
  args.vq = deferred_verify(p) ? p->rs.vq : nullptr;
  args.vq_len = p->rs.vq_len;
  args.vq_cap = p->rs.vq_cap;
  args.pos_leaf = p->rs.pos_leaf;
  args.perturb = p->opt.defer_test;
  args.katoms = (p->v.P + 31) / 32;
  args.prefetch = p->opt.l2_prefetch;
  args.trace = (a.depth == g_ws_trace_level) ? g_ws_trace : nullptr;
  args.spans = g_level_spans ? g_level_spans + (size_t)a.depth * kSMs * 4 : nullptr;
  auto launch = [&](auto kernel, size_t tables, int threads) -> int {
    const size_t smem = 1024 + ws2::kStages * ws2::kStageBytes + ws2::kBBytes + tables;
    FEPLL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (p->opt.pdl)
      FEPLL_CUDA(launch_pdl(kernel, dim3(kSMs), dim3(threads), smem, st, p->v, args));
    else
      kernel<<<kSMs, threads, smem, st>>>(p->v, args);
    return kOk;
  };
  if (p->level_tc_npad[a.depth] <= 96)
    launch(ws2::select_level_ws2_kernel<4, 96, 4, true>, sizeof(ws2::Smem<4>), ws2::threads_for(4, 4, true));
  else
    launch(ws2::select_level_ws2_kernel<3, 128, 4, false>, sizeof(ws2::Smem<3>), ws2::threads_for(3, 4, false));
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll

extern "C" int fepll_debug_level_spans(void* device_buffer) {
  fepll::g_level_spans = static_cast<uint64_t*>(device_buffer);
  return 0;
}
