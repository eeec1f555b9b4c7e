// Kernel (b), tensor-core path, deep-staging variant of select_ws.cu (P <= 64).
//
// Same arithmetic and routing as select_ws.cu (3xTF32 tcgen05 scoring of one
// tree level, certified argmin, FP64 re-scoring of the rest;
// pkg/src/fepll/tree.py:416-428, pkg/src/fepll/gmm.py:323-339); the operand
// staging differs:
//
//   * tcgen05 kind::tf32 reads only the top 19 bits of an FP32 operand
//     (truncation, tools/tf32_trunc_test.cu), so the raw FP32 patch row is
//     the hi operand as is.  Rows land by cp.async in one of four 32 KB
//     raw stages — three tiles of loads in flight, no register staging;
//   * only lo = z - trunc(z) is computed (per producer thread: one 128-byte
//     K atom of one row) and written to tensor memory with tcgen05.st; the
//     lo x B_hi pass takes its A operand from TMEM (two 64-column lo
//     buffers), hi x B_hi and hi x B_lo read the raw stage;
//   * three 128-column TMEM accumulators / epilogue groups (512 columns in
//     all with the lo buffers).
//
// Error budget of the split (tc_epi.cuh): |lo| < 2^-10 |z|, its TF32
// truncation error < 2^-20 |z|; with B's RNE split and the FP32 accumulation
// the projection stays within the 2^-18 ||z|| the guard assumes.
#include <algorithm>

#include "route.cuh"
#include "tc.cuh"
#include "tc_epi.cuh"

namespace fepll {

namespace ws2 {
constexpr int kRows = 128;
constexpr int kProducerWarps = 8;       // warp w: K atom w/4, TMEM lane quarter w%4
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;
// epilogue groups (== TMEM accumulators) and accumulator width are template
// parameters: <3, 128> for levels with nodes up to 128 padded columns,
// <4, 96> where every node fits 96 (four groups keep up with the MMAs)
constexpr int threads_for(int ng) { return (9 + 4 * ng) * 32; }
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

constexpr int kIdxAhead = 8;   // tiles of row indices in flight (>= 2 * kStages)
constexpr int kIdxRing = 9;
constexpr int kRawAhead = kStages - 1;  // raw loads issued this many tiles ahead

template <int NG>
struct Smem {
  int32_t idx_ring[2][kIdxRing][kRows];  // [K atom][slot][row]
  WsLevelTables lv;
  int64_t nd_off[kMaxNodes];      // segment offset of each depth-d node (a.off)
  int16_t nd_npad[kMaxNodes];     // padded group width
  int16_t nd_nk[kMaxNodes];       // child count
  EpiGroup epi[NG];
  uint64_t raw_empty[kStages], lo_full[kLoBufs], lo_empty[kLoBufs];
  uint64_t acc_full[NG], acc_empty[NG];
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
  uint64_t* trace;       // debug timeline: [CTA][64 tiles][8] clock64 stamps (or NULL)
};

__device__ __forceinline__ void stamp(const Args& a, int i, int slot) {
  if (a.trace && i < 64) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles (per-CTA relative timing)
    a.trace[((size_t)blockIdx.x * 64 + i) * 8 + slot] = t;
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

template <int NG, int ACC>
__global__ void __launch_bounds__(threads_for(NG), 1)
select_level_ws2_kernel(PlanView pv, Args args) {
  constexpr int kGroups = NG;
  constexpr int kAcc = ACC;                          // accumulator columns (>= node width)
  constexpr uint32_t kLoCol0 = NG * ACC;             // TMEM column of lo buffer 0
  static_assert(NG * ACC + kLoBufs * 64 <= 512, "TMEM: accumulators + lo buffers");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = tc::align1024(smem_raw);
  uint8_t* stageA = base;
  uint8_t* bbuf = base + kStages * kStageBytes;   // resident B (hi then lo)
  Smem<NG>& s = *reinterpret_cast<Smem<NG>*>(bbuf + kBBytes);
  const LevelArgs& a = args.a;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (warp == kMmaWarp) tc::tmem_alloc(&s.tmem_base, kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) tc::mbar_init(&s.raw_empty[i], 1);
    for (int i = 0; i < kLoBufs; ++i) {
      tc::mbar_init(&s.lo_full[i], kProducerWarps);
      tc::mbar_init(&s.lo_empty[i], 1);
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
    // thread = one 128-byte K atom of one row; warp w: atom w/4, TMEM lane
    // quarter w%4 (rows 32*(w%4) .. +31)
    const int row = tid & (kRows - 1);
    const int ka = warp >> 2;
    const bool active = ka < args.katoms;
    const int r8 = row & 7;
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    int32_t* ring = s.idx_ring[ka][0];
    auto issue_idx = [&](int j) {  // patch index of this row of tile j -> ring
      if (j < ntile) {
        const TileInfo ti = tile_info(a, s.lv, t_begin + j);
        int32_t* dst = ring + (j % kIdxRing) * kRows + row;
        if (row < ti.m) tc::cp_async4(dst, a.seg_in + s.nd_off[ti.k] + ti.first + row);
        else *dst = -1;
      }
    };
    // raw K atom of the warp's 32 rows of tile j -> stage j % kStages.  Each
    // instruction moves four whole 128-byte row atoms (lanes 8r..8r+7: the
    // 16-byte chunks of one row), so every request is a full line; the
    // indices come from the ring entries other lanes fetched (landed and
    // made warp-visible by the wait + __syncwarp of an earlier iteration).
    const int c16 = lane & 7;
    auto issue_raw = [&](int j) {
      if (j < ntile && active) {
        const int* rg = ring + (j % kIdxRing) * kRows + 32 * (warp & 3);
        uint8_t* stg = stageA + (j % kStages) * kStageBytes + ka * kAtomA + (warp & 3) * 4096;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = 4 * q + (lane >> 3);  // row inside the warp's 32
          const int g = rg[r];
          uint8_t* dst = stg + (r >> 3) * 1024 + (r & 7) * 128 + ((c16 ^ (r & 7)) << 4);
          if (g >= 0) tc::cp_async16(dst, args.Z32 + (int64_t)g * args.z32_pitch + ka * 32 + 4 * c16);
          else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    // prologue: indices of the first kIdxAhead tiles (one group, waited),
    // then raw rows of tiles 0 .. kRawAhead-1 (one group each)
    for (int j = 0; j < kIdxAhead; ++j) issue_idx(j);
    tc::cp_async_commit();
    tc::cp_async_wait<0>();
    __syncwarp();
    for (int j = 0; j < kRawAhead; ++j) {
      issue_raw(j);
      tc::cp_async_commit();
    }
    // iteration i commits one group {idx(i + kIdxAhead), raw(i + kRawAhead)};
    // raw(i) then always has exactly kRawAhead - 1 younger groups
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages, lb = i % kLoBufs;
      tc::cp_async_wait<kRawAhead - 1>();  // raw(i) (and idx through i + kIdxAhead - kRawAhead) landed
      __syncwarp();                         // ... including the lanes' parts of this thread's row
      if (tid == 0) stamp(args, i, 0);
      // lo = z - trunc(z) of this row's K atom -> TMEM lo buffer lb
      if (i >= kLoBufs) tc::mbar_wait(&s.lo_empty[lb], ((i / kLoBufs) - 1) & 1);
      tc::fence_after_sync();
      if (active) {
        const uint8_t* src = stageA + st * kStageBytes + ka * kAtomA + (row >> 3) * 1024 + r8 * 128;
        uint32_t lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = *reinterpret_cast<const float4*>(src + ((c ^ r8) << 4));
          lo[4 * c + 0] = __float_as_uint(x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u));
          lo[4 * c + 1] = __float_as_uint(x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u));
          lo[4 * c + 2] = __float_as_uint(x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u));
          lo[4 * c + 3] = __float_as_uint(x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u));
        }
        tc::tmem_st32(tmem + lane_off + kLoCol0 + lb * 64 + ka * 32, lo);
        tc::tmem_st_wait();
      }
      tc::fence_proxy_async_smem();  // the raw stage (cp.async writes) for the MMAs
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.lo_full[lb]);
      if (tid == 0) stamp(args, i, 1);
      // refill: tile i + kRawAhead into the stage tile i - 1 used
      const int nx = i + kRawAhead;
      if (nx < ntile && nx >= kStages)
        tc::mbar_wait(&s.raw_empty[nx % kStages], ((nx / kStages) - 1) & 1);
      issue_idx(i + kIdxAhead);
      issue_raw(nx);
      tc::cp_async_commit();
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

      const int lb = i % kLoBufs;
      tc::mbar_wait(&s.lo_full[lb], (i / kLoBufs) & 1);
      tc::fence_after_sync();
      if (lane == 0) stamp(args, i, 2);
      const uint32_t idesc = tc::idesc_tf32(kRows, npad);
      const uint32_t d = tmem + ac * kAcc;
      // descriptor start-address field counts 16-byte units
      const uint64_t A0 = a_base + (uint64_t)((st * kStageBytes) >> 4);
      for (int kq = 0; kq < args.katoms; ++kq) {
        const uint64_t a_hi = A0 + (uint64_t)((kq * kAtomA) >> 4);   // raw rows
        const uint32_t a_lo = tmem + kLoCol0 + lb * 64 + kq * 32;     // TMEM lo
        const uint64_t b_hi = b_base + (uint64_t)((kq * npad * 128) >> 4);
        const uint64_t b_lo = b_base + (uint64_t)((bhalf + kq * npad * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ko = 2 * kk;  // 8 tf32 = 32 bytes inside the swizzle atom
          const uint32_t acc = (kq > 0 || kk > 0) ? 1u : 0u;
          tc::mma_tf32_tmemA_warp(d, a_lo + 8 * kk, b_hi + ko, idesc, acc);
          tc::mma_tf32_warp(d, a_hi + ko, b_lo + ko, idesc, 1u);
          tc::mma_tf32_warp(d, a_hi + ko, b_hi + ko, idesc, 1u);
        }
      }
      tc::mma_commit_warp(&s.raw_empty[st]);
      tc::mma_commit_warp(&s.lo_empty[lb]);
      tc::mma_commit_warp(&s.acc_full[ac]);
      if (lane == 0) stamp(args, i, 3);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - kEpiWarp0;       // 0..11
    const int grp = ew >> 2;               // tiles with i % kGroups == grp
    const int row = 32 * (warp & 3) + lane;
    const uint32_t d_acc = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + grp * kAcc;
    EpiGroup& E = s.epi[grp];
    const int etid = (ew & 3) * 32 + lane;  // 0..127 inside the group
    const int bar_id = 1 + grp;
    const double guard = args.guard;
    // pending (previous tile's) route of this thread's row
    bool p_valid = false;
    int p_kind = 0, p_key = 0, p_lrank = 0, p_g = 0, p_u = 0, p_leaf = 0;
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
      } else {
        a.leafseg[p_b0 + slot] = p_g;
        a.labels[p_g] = p_leaf;
      }
    };
    for (int i = grp; i < ntile; i += kGroups, ++it) {
      const int cb = it % 3, pb = (it + 2) % 3, nb = (it + 1) % 3;
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
      // previous tile's reservations land in bbase[pb]; next buffer zeroed
      if (res_key >= 0) E.bbase[pb][res_key] = res;
      if (etid <= kMaxChildren) E.bcnt[nb][etid] = 0;
      // warp-aggregated local ranks of this tile's rows per key
      const int key = valid ? (flagged ? kMaxChildren : bi) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(peers) - 1;
      int wbase = 0;
      if (key >= 0 && lane == leader) wbase = atomicAdd(&E.bcnt[cb][key], __popc(peers));
      wbase = __shfl_sync(0xffffffffu, wbase, leader);
      const int lrank = wbase + __popc(peers & ((1u << lane) - 1u));
      named_bar(bar_id, 128);  // counts of this tile complete, bases of the previous visible
      // reserve this tile's segment ranges (results used next iteration)
      res_key = -1;
      if (etid < nk && E.bcnt[cb][etid] > 0) {
        res = atomicAdd(&a.cnt[E.ch.bfs[etid]], E.bcnt[cb][etid]);
        res_key = etid;
      } else if (etid == 127 && E.bcnt[cb][kMaxChildren] > 0) {
        res = atomicAdd(&args.queue_len[a.depth], E.bcnt[cb][kMaxChildren]);
        res_key = kMaxChildren;
      }
      // write the previous tile's rows
      flush(pb);
      // this tile's row becomes pending
      p_valid = valid;
      if (valid) {
        p_key = key;
        p_lrank = lrank;
        p_g = g;
        p_u = u;
        if (key == kMaxChildren) {
          p_kind = 0;
        } else {
          const int v = E.ch.bfs[key];
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
  if (warp == kMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace ws2


extern uint64_t* g_ws_trace;
extern int g_ws_trace_level;

int select_level_ws2(Plan* p, const LevelArgs& a, const float* Z32, const double* sq, double guard,
                     cudaStream_t st) {
  ws2::Args args;
  args.a = a;
  args.Z32 = Z32;
  args.z32_pitch = (p->v.P + 31) / 32 * 32;
  args.sq = sq;
  args.guard = guard > 0 ? guard : kDefaultGuard;
  args.queue = p->rs.queue;
  args.queue_len = p->rs.queue_len;
  args.katoms = (p->v.P + 31) / 32;
  args.trace = (a.depth == g_ws_trace_level) ? g_ws_trace : nullptr;
  auto launch = [&](auto kernel, size_t tables, int threads) -> int {
    const size_t smem = 1024 + ws2::kStages * ws2::kStageBytes + ws2::kBBytes + tables;
    FEPLL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kernel<<<kSMs, threads, smem, st>>>(p->v, args);
    return kOk;
  };
  if (p->level_tc_npad[a.depth] <= 96)
    launch(ws2::select_level_ws2_kernel<4, 96>, sizeof(ws2::Smem<4>), ws2::threads_for(4));
  else
    launch(ws2::select_level_ws2_kernel<3, 128>, sizeof(ws2::Smem<3>), ws2::threads_for(3));
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll

