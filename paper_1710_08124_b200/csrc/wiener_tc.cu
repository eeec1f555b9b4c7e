// Kernel (c), tensor-core form: Wiener estimates on tcgen05 with 3xTF32
// products (P <= 64, P % 16 == 0, ranks <= 64; plan option wiener_tc, the
// FP32-state mode's Wiener step).
//
// Restates pkg/src/fepll/gmm.py:352-359 for every patch of a leaf bucket
// (the grouping of pkg/src/fepll/solver.py:233-241):
//     C    = (Z U_k) * (gamma - gamma_tail)        128 x r
//     Zhat = C U_k^T + gamma_tail Z                128 x P
// and writes Zhat + dc (`vals = est + dc`, pkg/src/fepll/patches.py:198-222).
//
// The FP64 DMMA kernel (wiener.cu) is bound by the FP64 pipe (1.44 ms per
// iteration at 64 x 1024^2, 37 TFLOP/s peak).  Here both products run on the
// 5th-generation tensor cores as 3xTF32 (a_hi b_hi + a_lo b_hi + a_hi b_lo,
// FP32 accumulation in tensor memory; the two terms that share a_hi run as
// one pass against [b_hi; b_lo] stacked along N and are added by the
// epilogue, so a tile is 24 MMAs instead of 36 at rank <= 32):
// the result carries ~2^-20 relative error per product instead of FP64's
// 2^-53, far inside the restoration's tolerance (RMSE <= 1e-3 on 0..255,
// tests/test_gpu_fp32_state.py), and the kernel becomes HBM-bound: 256 B of
// FP32 row in, P x sizeof(OT) out per patch.
//
// One CTA per SM walks a contiguous range of 128-patch tiles in leaf order.
// Warp roles (22 warps):
//   0-3   loaders: the tile's FP32 rows by cp.async into one of NS 32 KB
//         stages, K-major 128B-swizzled (the layout tcgen05 reads); row
//         indices arrive a few tiles earlier in a ring;
//   4-7   converters: z_lo = z - trunc_tf32(z) into tensor memory (the
//         tensor core truncates FP32 operands to TF32, tools/
//         tf32_trunc_test.cu, so the raw row is z_hi as is);
//   8     first product issuer (the leaf's basis image arrives by one TMA
//         bulk copy when the leaf changes, 2-3 times per CTA per launch);
//   21    second product issuer (its own warp: a tile's second product
//         goes out as soon as its W is ready);
//   9-12  first epilogue: C (TMEM) * shrink -> W, W_lo = W - trunc(W), both
//         back into tensor memory as the second product's A operand;
//   13-20 second epilogue, two groups (one per TMEM set): Zhat = acc +
//         gamma_tail z (z from the raw stage) + dc, staged per warp in
//         shared memory and written as whole 256-byte row pieces (one TMA
//         bulk store per piece measured the same: 2.69 vs 2.64 ms/step).
// Tensor memory, two sets of 256 columns: [0,64) z_lo then W_lo, [64,128) C
// ([Z b_hi | Z b_lo] halves at rank <= 32) then W (in place), [128,256) the
// Zhat accumulator halves [W b_hi | W b_lo].
#include <algorithm>
#include <type_traits>

#include "route.cuh"
#include "tc.cuh"
#include "tc_epi.cuh"

namespace fepll {

namespace wtc {

constexpr int kRows = 128;
constexpr int kLoaderWarps = 4;                  // 32 rows each (two measured slower: the loaders became the limit)
constexpr int kLoaderRows = kRows / kLoaderWarps;
constexpr int kLoaderQ = kLoaderRows / 4;        // rows per lane (4 rows per instruction)
constexpr int kLoaderThreads = 32 * kLoaderWarps;
constexpr int kConvWarp0 = kLoaderWarps;
constexpr int kMmaWarp = kConvWarp0 + 4;
constexpr int kEp1Warp0 = kMmaWarp + 1;
constexpr int kEp2Warp0 = kEp1Warp0 + 4;
constexpr int kMma2Warp = kEp2Warp0 + 8;        // second product issuer
constexpr int kThreads = (kMma2Warp + 1) * 32;  // 704 (79 registers, no spills)
constexpr int kAtomA = kRows * 128;              // bytes of one K atom of a row stage
constexpr int kStageBytes = 2 * kAtomA;          // P <= 64: two K atoms
constexpr int kMaxR = 64;
template <class OT>
constexpr int unit_cols() { return 256 / (int)sizeof(OT); }  // columns per staged 256-byte output piece
template <class OT>
constexpr int out_pitch() { return 256 + 16; }  // +16: conflict-free 16-byte stores
constexpr int kIdxAhead = 4;
constexpr int kSwitchCost = 3;                   // tiles' worth of time a leaf switch costs (CTA split)
constexpr int kMaxStages = 4;
constexpr int kIdxRing = kMaxStages + kIdxAhead + 2;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kSetCols = 256;               // TMEM columns between the two sets
constexpr uint32_t kColLo = 0, kColC = 64, kColOut = 128;

struct Smem {
  int32_t idx_ring[kIdxRing][kRows];
  int32_t tpre[kMaxLevelNodes + 1];
  uint64_t scan_tmp[256];
  int32_t leaf_cr[kMaxLevelNodes];   // component | rank << 16
  int32_t leaf_cnt[kMaxLevelNodes];
  float leaf_gt[kMaxLevelNodes];     // gamma_tail at this iteration
  int64_t leaf_off[kMaxLevelNodes];
  float shrink[kMaxR];               // first epilogue: the current leaf's gamma - gamma_tail
  uint64_t raw_full[kMaxStages], stage_free[kMaxStages];
  uint64_t lo_full[2], c_full[2], w_full[2], out_full[2], out_empty[2];
  uint64_t drain, b_full, drain2, b2_full;
  uint32_t tmem_base;
  int32_t t_begin, t_end;
};

struct Args {
  int t;
  const int32_t* leaf_nodes;
  int n_leaf_nodes;
  const int32_t* cnt;
  const int64_t* off;
  const int32_t* leafseg;
  const float* Z32;
  int z32_pitch;
  const double* dc;
  void* Zhat;
  int n_img, zrows;
  int P, katoms, ns;
  int bq1, bq2;        // bytes of the first / second product's basis image ([hi rows; lo rows] per K atom)
  const uint8_t* img;  // [K][bq1 + bq2] the components' basis images (basis_images_kernel)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float trunc_tf32(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// debug profile (fepll_debug_wtc_prof): [CTA][32] cycles spent in each role's
// waits, accumulated by the role's first lane
__device__ uint64_t* g_prof = nullptr;
#ifdef FEPLL_WTC_PROF
struct Prof {
  uint64_t* out;
  bool on;
  uint64_t acc[4] = {0, 0, 0, 0};
  __device__ __forceinline__ Prof(bool leader) {
    out = g_prof;
    on = out != nullptr && leader;
  }
  __device__ __forceinline__ uint64_t now() const {
    uint64_t t = 0;
    if (on) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
  }
  __device__ __forceinline__ void add(int k, uint64_t t0) {
    if (on) acc[k] += now() - t0;
  }
  __device__ __forceinline__ void flush(int slot0, int n) {
    if (on)
      for (int k = 0; k < n; ++k) out[(size_t)blockIdx.x * 32 + slot0 + k] = acc[k];
  }
};
#else
// compiled out by default (build with -DFEPLL_WTC_PROF, tools/wtc_prof.py): the
// counters cost the epilogue roles registers
struct Prof {
  static constexpr bool on = false;
  uint64_t* out = nullptr;
  uint64_t acc[4] = {0, 0, 0, 0};
  __device__ __forceinline__ Prof(bool) {}
  __device__ __forceinline__ uint64_t now() const { return 0; }
  __device__ __forceinline__ void add(int, uint64_t) {}
  __device__ __forceinline__ void flush(int, int) {}
};
#endif

// tile -> leaf (index into the leaf tables); tiles ascend
struct LeafCursor {
  int k = -1;
  __device__ __forceinline__ int at(const Smem& s, int n, int tile) {
    if (k < 0) k = prefix_find(s.tpre, n, tile);
    while (k + 1 < n && s.tpre[k + 1] <= tile) ++k;
    return k;
  }
};

template <class OT>
__global__ void __launch_bounds__(kThreads, 1) wiener_tc_kernel(PlanView pv, Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = tc::align1024(smem_raw);
  const int NS = a.ns;
  uint8_t* stageA = base;
  uint8_t* bbuf = base + NS * kStageBytes;           // B1 (a.bq1 bytes), B2 (a.bq2 bytes)
  uint8_t* outbuf = bbuf + a.bq1 + a.bq2;            // [8 warps][32 rows][kOutPitch]
  constexpr int kOutPitch = out_pitch<OT>();
  constexpr int kUnitCols = unit_cols<OT>();
  Smem& s = *reinterpret_cast<Smem*>(outbuf + 8 * 32 * kOutPitch);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nl = a.n_leaf_nodes;
  const int P = a.P;

  if (warp == kMmaWarp) tc::tmem_alloc(&s.tmem_base, kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < kMaxStages; ++i) {
      tc::mbar_init(&s.raw_full[i], kLoaderThreads);
      tc::mbar_init(&s.stage_free[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.lo_full[i], 4);
      tc::mbar_init(&s.c_full[i], 1);
      tc::mbar_init(&s.w_full[i], 4);
      tc::mbar_init(&s.out_full[i], 1);
      tc::mbar_init(&s.out_empty[i], 4);
    }
    tc::mbar_init(&s.drain, 1);
    tc::mbar_init(&s.b_full, 1);
    tc::mbar_init(&s.drain2, 1);
    tc::mbar_init(&s.b2_full, 1);
    tc::fence_mbar_init();
  }
  for (int k = tid; k < nl; k += kThreads) {
    const int v = a.leaf_nodes[k];
    const int comp = pv.leaf_index[v];
    s.leaf_cr[k] = comp | (pv.model_rank[comp] << 16);
    s.leaf_gt[k] = (float)pv.model_gamma_tail[(int64_t)a.t * pv.K + comp];
    s.leaf_cnt[k] = a.cnt[v];
    s.leaf_off[k] = a.off[v];
    s.tpre[k] = (a.cnt[v] + kRows - 1) / kRows;
  }
  __syncthreads();
  const int tiles = block_exscan(s.tpre, nl, s.scan_tmp);
  if (tid == 0) {
    s.tpre[nl] = tiles;
    // contiguous tile ranges of equal estimated cost: a tile costs 1, every
    // leaf entered kSwitchCost more (its basis images are loaded while the
    // tensor pipe drains) — the small leaves would otherwise leave the CTAs
    // holding many of them behind
    int nz = 0;
    for (int k = 0; k < nl; ++k) nz += s.tpre[k + 1] > s.tpre[k];
    const int64_t Wt = (int64_t)tiles + (int64_t)kSwitchCost * nz;
    const int64_t x0 = Wt * blockIdx.x / gridDim.x, x1 = Wt * (blockIdx.x + 1) / gridDim.x;
    int64_t acc = 0;
    int tb = tiles, te = tiles;
    for (int k = 0; k < nl; ++k) {
      const int nt = s.tpre[k + 1] - s.tpre[k];
      if (nt == 0) continue;
      // tile j of this leaf ends at cost acc + kSwitchCost + j + 1
      const int64_t lo = acc + kSwitchCost, nxt = lo + nt;
      if (tb == tiles && x0 < nxt) tb = s.tpre[k] + (int)max((int64_t)0, x0 - lo);
      if (te == tiles && x1 < nxt) te = s.tpre[k] + (int)max((int64_t)0, x1 - lo);
      acc = nxt;
    }
    s.t_begin = blockIdx.x == 0 ? 0 : tb;
    s.t_end = blockIdx.x + 1 == gridDim.x ? tiles : te;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s.tmem_base;
  const int t_begin = s.t_begin, t_end = s.t_end;
  const int ntile = t_end - t_begin;
  const int64_t pitch = a.z32_pitch;

  if (warp < kLoaderWarps) {
    // ------------------------------------------------------------ loaders
    const int r0 = kLoaderRows * warp;
    LeafCursor cur;
    auto issue_idx = [&](int j) {
      if (j < ntile) {
        const int li = cur.at(s, nl, t_begin + j);
        const int first = (t_begin + j - s.tpre[li]) * kRows;
        int32_t* ring = s.idx_ring[j % kIdxRing];
#pragma unroll
        for (int h = 0; h < kLoaderRows / 32; ++h) {
          const int row = r0 + 32 * h + lane;
          if (row < s.leaf_cnt[li] - first) tc::cp_async4(ring + row, a.leafseg + s.leaf_off[li] + first + row);
          else ring[row] = -1;
        }
      }
    };
    const int c16 = lane & 7;
    Prof pf(tid == 0);
    const uint64_t tl0 = pf.now();
    for (int j = 0; j < kIdxAhead; ++j) {
      issue_idx(j);
      tc::cp_async_commit();
    }
    for (int i = 0; i < ntile; ++i) {
      const int st = i % NS;
      const uint64_t tw = pf.now();
      if (i >= NS) tc::mbar_wait(&s.stage_free[st], ((i / NS) - 1) & 1);
      pf.add(0, tw);
      tc::cp_async_wait<kIdxAhead - 1>();  // idx(i) landed (one group per tile)
      __syncwarp();
      const int32_t* rg = s.idx_ring[i % kIdxRing] + r0;
      int g[kLoaderQ];
#pragma unroll
      for (int q = 0; q < kLoaderQ; ++q) g[q] = rg[4 * q + (lane >> 3)];
      uint8_t* stg = stageA + st * kStageBytes + (r0 >> 3) * 1024;
#pragma unroll
      for (int ka = 0; ka < 2; ++ka) {
        if (ka < a.katoms) {
          const float* zb = a.Z32 + ka * 32 + 4 * c16;
#pragma unroll
          for (int q = 0; q < kLoaderQ; ++q) {
            const int r = 4 * q + (lane >> 3);
            uint8_t* dst = stg + ka * kAtomA + (r >> 3) * 1024 + (r & 7) * 128 + ((c16 ^ (r & 7)) << 4);
            // holes and rows past the bucket's end land as zeros (no bytes read)
            tc::cp_async16_zfill(dst, g[q] >= 0 ? zb + g[q] * pitch : a.Z32, g[q] >= 0 ? 16u : 0u);
          }
        }
      }
      issue_idx(i + kIdxAhead);
      tc::cp_async_commit();
      tc::cp_async_mbar_arrive(&s.raw_full[st]);
    }
    tc::cp_async_wait<0>();
    pf.add(1, tl0);
    pf.flush(0, 2);  // [0] stage_free wait, [1] loader loop total
  } else if (warp < kMmaWarp) {
    // ------------------------------------------------------------ converters
    const int quarter = warp & 3;
    const int row = 32 * quarter + lane;
    const int r8 = row & 7;
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    Prof pf(warp == kConvWarp0 && lane == 0);
    const uint64_t tl0 = pf.now();
    for (int i = 0; i < ntile; ++i) {
      const int st = i % NS, set = i & 1;
      uint64_t tw = pf.now();
      tc::mbar_wait(&s.raw_full[st], (i / NS) & 1);
      pf.add(0, tw);
      tw = pf.now();
      // the set's z_lo / W_lo columns: tile i - 2's second product has read them
      if (i >= 2) tc::mbar_wait(&s.out_full[set], ((i - 2) >> 1) & 1);
      pf.add(1, tw);
      tc::fence_after_sync();
      const uint32_t xb = tmem + lane_off + set * kSetCols + kColLo;
      for (int ka = 0; ka < a.katoms; ++ka) {
        const uint8_t* src = stageA + st * kStageBytes + ka * kAtomA + (row >> 3) * 1024 + r8 * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t xl[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 x = *reinterpret_cast<const float4*>(src + (((4 * h + c) ^ r8) << 4));
            xl[4 * c] = __float_as_uint(x.x - trunc_tf32(x.x));  // exact differences
            xl[4 * c + 1] = __float_as_uint(x.y - trunc_tf32(x.y));
            xl[4 * c + 2] = __float_as_uint(x.z - trunc_tf32(x.z));
            xl[4 * c + 3] = __float_as_uint(x.w - trunc_tf32(x.w));
          }
          tc::tmem_st16(xb + 32 * ka + 16 * h, xl);
        }
      }
      tc::tmem_st_wait();
      tc::fence_proxy_async_smem();  // the landed raw stage, for the MMAs' async-proxy reads
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.lo_full[set]);
    }
    pf.add(2, tl0);
    pf.flush(2, 3);  // [2] raw_full wait, [3] out_full wait, [4] converter loop total
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ first product issuer
    // The whole warp runs this loop (uniform values); one elected lane
    // issues each tcgen05 instruction (tc.cuh *_warp).
    const uint64_t a_base = tc::desc_sw128(tc::smem_u32(stageA));
    const uint64_t d_b1 = tc::desc_sw128(tc::smem_u32(bbuf));
    LeafCursor cur;
    int cur_leaf = -1, R = 16;
    uint32_t drains = 0, b_loads = 0;
    Prof pf(lane == 0);
    Prof pf2(lane == 0);
    const uint64_t tl0 = pf.now();
    for (int i = 0; i < ntile; ++i) {
      const int st = i % NS, set = i & 1;
      const int li = cur.at(s, nl, t_begin + i);
      if (li != cur_leaf) {
        const uint64_t tb = pf2.now();
        if (i > 0) {  // the previous tiles' first products still read the old image
          tc::mma_commit_warp(&s.drain);
          tc::mbar_wait(&s.drain, drains & 1);
          ++drains;
        }
        const int comp = s.leaf_cr[li] & 0xFFFF, r = s.leaf_cr[li] >> 16;
        R = max(16, (r + 15) & ~15);
        if (lane == 0) {
          tc::mbar_arrive_expect_tx(&s.b_full, (uint32_t)a.bq1);
          tc::bulk_g2s(bbuf, a.img + (size_t)comp * (a.bq1 + a.bq2), (uint32_t)a.bq1, &s.b_full);
        }
        __syncwarp();
        tc::mbar_wait(&s.b_full, b_loads & 1);
        ++b_loads;
        cur_leaf = li;
        pf2.add(0, tb);
      }
      // first product of tile i (K = 32 katoms): C = Z [B1_hi; B1_lo], C[0,R) += Z_lo B1_hi.
      // The passes that read Z from the raw stage start as soon as the rows
      // land and the set's C columns are free (tile i - 2's second product has
      // read W there); the Z_lo pass follows once the converters are done.
      uint64_t tw = pf.now();
      tc::mbar_wait(&s.raw_full[st], (i / NS) & 1);
      if (i >= 2) tc::mbar_wait(&s.out_full[set], ((i - 2) >> 1) & 1);
      pf.add(0, tw);
      tc::fence_after_sync();
      tc::fence_proxy_async_smem();
      {
        const uint64_t tg = pf2.now();
        const uint32_t d = tmem + set * kSetCols + kColC;
        const uint32_t z_lo = tmem + set * kSetCols + kColLo;
        const uint32_t idesc = tc::idesc_tf32(kRows, R);
        const uint64_t A0 = a_base + (uint64_t)((st * kStageBytes) >> 4);
        const uint64_t rstep = (uint64_t)((2 * R * 128) >> 4);  // B1 atom stride ([hi; lo] rows)
        const uint64_t lo_rows = (uint64_t)((R * 128) >> 4);    // the lo rows inside an atom
        if (R <= 32) {
          // Z (smem, read as trunc_tf32) . [B1_hi; B1_lo] (both halves in one pass) alternating with
          // Z_lo (TMEM) . B1_hi: a run of TMEM-operand MMAs alone issues at ~131 cycles each, one
          // between two shared-memory-operand MMAs at ~50 (tools/mma_bench.cu, Wiener tile patterns)
          const uint32_t idescw = tc::idesc_tf32(kRows, 2 * R);
          tw = pf.now();
          tc::mbar_wait(&s.lo_full[set], (i >> 1) & 1);
          pf.add(1, tw);
          tc::fence_after_sync();
          for (int kq = 0; kq < a.katoms; ++kq) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              tc::mma_tf32_warp(d, A0 + (uint64_t)(kq * (kAtomA >> 4) + 2 * kk), d_b1 + kq * rstep + 2 * kk,
                                idescw, (kq > 0 || kk > 0) ? 1u : 0u);
              tc::mma_tf32_tmemA_warp(d, z_lo + 32 * kq + 8 * kk, d_b1 + kq * rstep + 2 * kk, idesc, 1u);
            }
          }
        } else {
          for (int kq = 0; kq < a.katoms; ++kq) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc::mma_tf32_warp(d, A0 + (uint64_t)(kq * (kAtomA >> 4) + 2 * kk), d_b1 + kq * rstep + 2 * kk, idesc,
                                (kq > 0 || kk > 0) ? 1u : 0u);
          }
          tw = pf.now();
          tc::mbar_wait(&s.lo_full[set], (i >> 1) & 1);
          pf.add(1, tw);
          tc::fence_after_sync();
          // Z . B1_lo alternating with Z_lo (TMEM) . B1_hi
          for (int kq = 0; kq < a.katoms; ++kq) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              tc::mma_tf32_warp(d, A0 + (uint64_t)(kq * (kAtomA >> 4) + 2 * kk),
                                d_b1 + lo_rows + kq * rstep + 2 * kk, idesc, 1u);
              tc::mma_tf32_tmemA_warp(d, z_lo + 32 * kq + 8 * kk, d_b1 + kq * rstep + 2 * kk, idesc, 1u);
            }
          }
        }
        tc::mma_commit_warp(&s.c_full[set]);
        pf2.add(2, tg);
      }
    }
    pf2.add(1, tl0);
    pf.flush(5, 2);   // [5] raw_full, [6] lo_full waits
    pf2.flush(9, 2);  // [9] leaf switches (drain + image load), [10] issuer loop total
    if (pf2.on) pf2.out[(size_t)blockIdx.x * 32 + 21] = pf2.acc[2];  // first product issue
  } else if (warp == kMma2Warp) {
    // ------------------------------------------------------------ second product issuer
    // its own warp: tile i's second product goes out as soon as the first
    // epilogue hands W over, not behind tile i + 1's first product
    const uint64_t d_b2 = tc::desc_sw128(tc::smem_u32(bbuf + a.bq1));
    const uint32_t idesc2w = tc::idesc_tf32(kRows, 2 * P), idesc2 = tc::idesc_tf32(kRows, P);
    LeafCursor cur;
    int cur_leaf = -1, R = 16;
    uint32_t drains = 0, b_loads = 0;
    Prof pf(lane == 0);
    const uint64_t tl0 = pf.now();
    for (int j = 0; j < ntile; ++j) {
      const int set = j & 1;
      const int li = cur.at(s, nl, t_begin + j);
      if (li != cur_leaf) {
        if (j > 0) {
          tc::mma_commit_warp(&s.drain2);
          tc::mbar_wait(&s.drain2, drains & 1);
          ++drains;
        }
        const int comp = s.leaf_cr[li] & 0xFFFF, r = s.leaf_cr[li] >> 16;
        R = max(16, (r + 15) & ~15);
        if (lane == 0) {
          tc::mbar_arrive_expect_tx(&s.b2_full, (uint32_t)a.bq2);
          tc::bulk_g2s(bbuf + a.bq1, a.img + (size_t)comp * (a.bq1 + a.bq2) + a.bq1, (uint32_t)a.bq2, &s.b2_full);
        }
        __syncwarp();
        tc::mbar_wait(&s.b2_full, b_loads & 1);
        ++b_loads;
        cur_leaf = li;
      }
      // second product of tile j (K = R): Out[0,2P) = W [B2_hi; B2_lo], Out[0,P) += W_lo B2_hi
      uint64_t tw = pf.now();
      tc::mbar_wait(&s.w_full[set], (j >> 1) & 1);
      pf.add(0, tw);
      tw = pf.now();
      if (j >= 2) tc::mbar_wait(&s.out_empty[set], ((j - 2) >> 1) & 1);
      pf.add(1, tw);
      tc::fence_after_sync();
      const uint64_t tg = pf.now();
      const uint32_t d = tmem + set * kSetCols + kColOut;
      const uint32_t w_hi = tmem + set * kSetCols + kColC, w_lo = tmem + set * kSetCols + kColLo;
      const int kpairs = R >> 4;  // R is a multiple of 16: two K steps per trip
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const uint32_t aw = pass == 1 ? w_lo : w_hi;
        const uint32_t id = pass == 1 ? idesc2 : idesc2w;
        for (int kp = 0; kp < kpairs; ++kp) {
          // K steps 2 kp, 2 kp + 1: atom kp / 2 (32 columns, 2P rows), 32-byte steps inside
          const uint64_t bo = (uint64_t)(((kp >> 1) * 2 * P * 128 + (kp & 1) * 64) >> 4);
          tc::mma_tf32_tmemA_warp(d, aw + 16 * kp, d_b2 + bo, id, (pass > 0 || kp > 0) ? 1u : 0u);
          tc::mma_tf32_tmemA_warp(d, aw + 16 * kp + 8, d_b2 + bo + 2, id, 1u);
        }
      }
      tc::mma_commit_warp(&s.out_full[set]);
      pf.add(2, tg);
    }
    pf.add(3, tl0);
    pf.flush(7, 2);  // [7] w_full, [8] out_empty waits
    if (pf.on) {
      pf.out[(size_t)blockIdx.x * 32 + 22] = pf.acc[2];  // second product issue
      pf.out[(size_t)blockIdx.x * 32 + 23] = pf.acc[3];  // its loop total
    }
  } else if (warp < kEp2Warp0) {
    // ------------------------------------------------------------ first epilogue
    const int quarter = warp & 3;
    const int etid = (warp - kEp1Warp0) * 32 + lane;
    const uint32_t lane_off = (uint32_t)(32 * quarter) << 16;
    LeafCursor cur;
    int my_leaf = -1;
    Prof pf(etid == 0);
    const uint64_t tl0 = pf.now();
    for (int i = 0; i < ntile; ++i) {
      const int set = i & 1;
      const int li = cur.at(s, nl, t_begin + i);
      const int comp = s.leaf_cr[li] & 0xFFFF, r = s.leaf_cr[li] >> 16;
      const int R = max(16, (r + 15) & ~15);
      if (li != my_leaf) {
        named_bar(1, 128);  // everyone done with the previous leaf's table
        const double* shrink = pv.model_shrink + (int64_t)a.t * pv.model_cols_total + pv.model_col_off[comp];
        if (etid < kMaxR) s.shrink[etid] = etid < r ? (float)shrink[etid] : 0.0f;
        my_leaf = li;
        named_bar(1, 128);
      }
      const uint64_t tw = pf.now();
      tc::mbar_wait(&s.c_full[set], (i >> 1) & 1);
      pf.add(0, tw);
      tc::fence_after_sync();
      const uint32_t cb = tmem + lane_off + set * kSetCols + kColC;
      const uint32_t lb = tmem + lane_off + set * kSetCols + kColLo;
      const bool wide = R <= 32;
      for (int c = 0; c < R; c += 16) {
        uint32_t w[16], wl[16];
        tmem_ld16(cb + c, w);
        if (wide) tmem_ld16(cb + R + c, wl);  // the Z B1_lo half
        tc::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float cv = wide ? __uint_as_float(w[k]) + __uint_as_float(wl[k]) : __uint_as_float(w[k]);
          const float v = cv * s.shrink[c + k];
          w[k] = __float_as_uint(v);  // read as trunc_tf32(v) by the tensor core
          wl[k] = __float_as_uint(v - trunc_tf32(v));
        }
        tc::tmem_st16(cb + c, w);
        tc::tmem_st16(lb + c, wl);
      }
      tc::tmem_st_wait();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.w_full[set]);
    }
    pf.add(1, tl0);
    pf.flush(11, 2);  // [11] c_full wait, [12] first-epilogue loop total
  } else {
    // ------------------------------------------------------------ second epilogue
    const int ew = warp - kEp2Warp0;   // 0..7
    const int grp = ew >> 2;           // == TMEM set
    const int quarter = warp & 3;
    const int row = 32 * quarter + lane;
    const int r8 = row & 7;
    const uint32_t d_acc = tmem + ((uint32_t)(32 * quarter) << 16) + grp * kSetCols + kColOut;
    uint8_t* ob = outbuf + ew * 32 * kOutPitch;  // this warp's 32 staged row pieces
    uint8_t* orow_s = ob + lane * kOutPitch;
    OT* Zhat = static_cast<OT*>(a.Zhat);
    LeafCursor cur;
    Prof pf((ew & 3) == 0 && lane == 0);
    const uint64_t tl0 = pf.now();
    for (int i = grp; i < ntile; i += 2) {
      const int st = i % NS;
      const int li = cur.at(s, nl, t_begin + i);
      const float gt = s.leaf_gt[li];
      const int32_t* ring = s.idx_ring[i % kIdxRing];
      // the tile's indices landed before its rows: dc is fetched while the
      // products run
      uint64_t tw = pf.now();
      tc::mbar_wait(&s.raw_full[st], (i / NS) & 1);
      pf.add(0, tw);
      const int g = ring[row];
      const double dcv = g >= 0 ? a.dc[g] : 0.0;
      const float dcf = (float)dcv;
      tw = pf.now();
      tc::mbar_wait(&s.out_full[grp], (i >> 1) & 1);
      pf.add(1, tw);
      tc::fence_after_sync();
      const uint64_t tc0 = pf.now();
      const uint8_t* zsrc = stageA + st * kStageBytes + (row >> 3) * 1024 + r8 * 128;
      for (int c0 = 0; c0 < P; c0 += kUnitCols) {
        const int ucols = min(kUnitCols, P - c0);
        for (int c = c0; c < c0 + ucols; c += 16) {
          uint32_t acc[16], acl[16];
          tmem_ld16(d_acc + c, acc);
          tmem_ld16(d_acc + P + c, acl);  // the W B2_lo half
          // z columns c .. c+15: atom c / 32, 16-byte chunks 4 (c/16 % 2) ..
          const uint8_t* za = zsrc + (c >> 5) * kAtomA;
          const int ch0 = ((c >> 4) & 1) * 4;
          float4 z[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) z[q] = *reinterpret_cast<const float4*>(za + (((ch0 + q) ^ r8) << 4));
          tc::tmem_ld_wait();
          OT* dst = reinterpret_cast<OT*>(orow_s) + (c - c0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float e0 = fmaf(gt, z[q].x, __uint_as_float(acc[4 * q]) + __uint_as_float(acl[4 * q]));
            const float e1 = fmaf(gt, z[q].y, __uint_as_float(acc[4 * q + 1]) + __uint_as_float(acl[4 * q + 1]));
            const float e2 = fmaf(gt, z[q].z, __uint_as_float(acc[4 * q + 2]) + __uint_as_float(acl[4 * q + 2]));
            const float e3 = fmaf(gt, z[q].w, __uint_as_float(acc[4 * q + 3]) + __uint_as_float(acl[4 * q + 3]));
            if constexpr (sizeof(OT) == 8) {
              const double o0 = (double)e0 + dcv, o1 = (double)e1 + dcv, o2 = (double)e2 + dcv,
                           o3 = (double)e3 + dcv;
              *reinterpret_cast<double2*>(dst + 4 * q) = make_double2(o0, o1);
              *reinterpret_cast<double2*>(dst + 4 * q + 2) = make_double2(o2, o3);
            } else {
              // FP32 rows: est + dc in FP32 (one more 2^-24 rounding next to the store's)
              *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(e0 + dcf, e1 + dcf, e2 + dcf, e3 + dcf);
            }
          }
        }
        const bool last = c0 + kUnitCols >= P;
        if (last) pf.add(2, tc0);
        if (last) {
          // accumulator and raw stage are read: release both
          tc::fence_before_sync();
        }
        __syncwarp();
        if (last && lane == 0) {
          mbar_arrive(&s.out_empty[grp]);
          mbar_arrive(&s.stage_free[st]);
        }
        const int ubytes = ucols * (int)sizeof(OT);
        // write the warp's 32 row pieces: kLpr lanes cover a piece (16 bytes each), 32 / kLpr rows per instruction
        constexpr int kLpr = kUnitCols * (int)sizeof(OT) / 16;
        const int hl = lane % kLpr;
#pragma unroll 4
        for (int rr = 0; rr < 32; rr += 32 / kLpr) {
          const int lr = rr + lane / kLpr;
          const int gg = ring[32 * quarter + lr];
          if (gg >= 0 && hl * 16 < ubytes) {
            const int64_t orow =
                a.zrows == a.n_img ? (int64_t)gg : (int64_t)(gg / a.n_img) * a.zrows + gg % a.n_img;
            const uint4 v = *reinterpret_cast<const uint4*>(ob + lr * kOutPitch + hl * 16);
            *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(Zhat + orow * P + c0) + hl * 16) = v;
          }
        }
        __syncwarp();  // the pieces are read before the next unit overwrites them
      }
    }
    pf.add(3, tl0);
    pf.flush(13 + 4 * grp, 4);  // [13/17] raw_full, [14/18] out_full waits, [15/19] compute, [16/20] loop total
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

// The components' basis images, built once per plan: for component k,
// R = its rank rounded up to 16, two images in the K-major 128B-swizzled
// layout tcgen05 reads, the hi rows followed by the lo rows in every K atom —
//   B1: rows j (rank) then R + j, K = p (patch element), atoms of 32 p;
//   B2: rows p then P + p, K = j, atoms of 32 j —
// hi = rna_tf32(u), lo = u - hi (FP32; the tensor core truncates it to TF32).
__global__ void basis_images_kernel(PlanView pv, int katoms, int bq1, int bq2, uint8_t* img) {
  const int comp = blockIdx.x;
  const int P = pv.P, r = pv.model_rank[comp];
  const int R = max(16, (r + 15) & ~15);
  const double* U = pv.model_basis + pv.model_off64[comp];  // [P][r]
  uint8_t* b1 = img + (size_t)comp * (bq1 + bq2);
  uint8_t* b2 = b1 + bq1;
  for (int e = threadIdx.x; e < (bq1 + bq2) / 4; e += blockDim.x) reinterpret_cast<float*>(b1)[e] = 0.0f;
  __syncthreads();
  auto at = [](int row, int k) {  // row inside an atom, k in [0, 32): 128B swizzle
    return (row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7))) << 4) + (k & 3) * 4;
  };
  const int KP = 32 * katoms;
  for (int e = threadIdx.x; e < KP * R; e += blockDim.x) {
    const int p = e / R, j = e - p * R;
    const float u = (p < P && j < r) ? (float)U[(int64_t)p * r + j] : 0.0f;
    const float hi = tc::to_tf32(u), lo = u - hi;
    uint8_t* a1 = b1 + (p >> 5) * (2 * R * 128);
    *reinterpret_cast<float*>(a1 + at(j, p & 31)) = hi;
    *reinterpret_cast<float*>(a1 + at(R + j, p & 31)) = lo;
    if (p < P) {
      uint8_t* a2 = b2 + (j >> 5) * (2 * P * 128);
      *reinterpret_cast<float*>(a2 + at(p, j & 31)) = hi;
      *reinterpret_cast<float*>(a2 + at(P + p, j & 31)) = lo;
    }
  }
}

}  // namespace wtc
}  // namespace fepll

extern "C" int fepll_debug_wtc_prof(void* device_buffer) {
  uint64_t* p = static_cast<uint64_t*>(device_buffer);
  return cudaMemcpyToSymbol(fepll::wtc::g_prof, &p, sizeof(p)) == cudaSuccess ? 0 : 5;
}

namespace fepll {

bool wiener_tc_supported(const Plan* p) {
  const int P = p->v.P;
  return P % 16 == 0 && P <= 64 && p->max_model_rank <= wtc::kMaxR && p->n_leaf_nodes <= kMaxLevelNodes;
}

static void wtc_image_bytes(const Plan* p, int* bq1, int* bq2) {
  const int katoms = (p->v.P + 31) / 32;
  const int rmax = std::max(16, (p->max_model_rank + 15) & ~15);
  *bq1 = katoms * 2 * rmax * 128;
  *bq2 = (rmax + 31) / 32 * 2 * p->v.P * 128;
}

// plan creation: the basis images of every component (K x (bq1 + bq2) bytes)
int wiener_tc_prepare(Plan* p) {
  if (!wiener_tc_supported(p)) return kOk;
  int bq1, bq2;
  wtc_image_bytes(p, &bq1, &bq2);
  void* m = nullptr;
  FEPLL_CUDA(cudaMalloc(&m, (size_t)p->v.K * (bq1 + bq2)));
  p->owned.push_back(m);
  p->wtc_img = static_cast<uint8_t*>(m);
  wtc::basis_images_kernel<<<p->v.K, 256>>>(p->v, (p->v.P + 31) / 32, bq1, bq2, p->wtc_img);
  FEPLL_LAUNCH();
  FEPLL_CUDA(cudaDeviceSynchronize());
  return kOk;
}

template <class OT>
static int wiener_tc_t(Plan* p, int t, const float* Z32, int z32_pitch, const double* dc, OT* Zhat, int n_img,
                       int zrows, cudaStream_t st) {
  wtc::Args a;
  a.t = t;
  a.leaf_nodes = p->d_leaf_nodes;
  a.n_leaf_nodes = p->n_leaf_nodes;
  a.cnt = p->rs.cnt;
  a.off = p->rs.off;
  a.leafseg = p->rs.leafseg;
  a.Z32 = Z32;
  a.z32_pitch = z32_pitch;
  a.dc = dc;
  a.Zhat = Zhat;
  a.n_img = n_img;
  a.zrows = zrows;
  a.P = p->v.P;
  a.katoms = (p->v.P + 31) / 32;
  wtc_image_bytes(p, &a.bq1, &a.bq2);
  a.img = p->wtc_img;
  FEPLL_REQUIRE(a.img != nullptr, "wiener_tc: the plan holds no basis images");
  int dev = 0, optin = 0;
  FEPLL_CUDA(cudaGetDevice(&dev));
  FEPLL_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  auto smem_for = [&](int ns) {
    return 1024 + (size_t)ns * wtc::kStageBytes + (size_t)(a.bq1 + a.bq2) + 8 * 32 * wtc::out_pitch<OT>() + sizeof(wtc::Smem);
  };
  a.ns = smem_for(4) <= (size_t)optin ? 4 : smem_for(3) <= (size_t)optin ? 3 : 2;
  const size_t smem = smem_for(a.ns);
  FEPLL_REQUIRE(smem <= (size_t)optin, "wiener_tc: tile buffers exceed shared memory");
  auto kernel = wtc::wiener_tc_kernel<OT>;
  FEPLL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kernel<<<kSMs, wtc::kThreads, smem, st>>>(p->v, a);
  FEPLL_LAUNCH();
  return kOk;
}

int wiener_tc_f32(Plan* p, int t, const float* Z32, int z32_pitch, const double* dc, float* Zhat, int n_img,
                  int zrows, cudaStream_t st) {
  return wiener_tc_t<float>(p, t, Z32, z32_pitch, dc, Zhat, n_img, zrows, st);
}

int wiener_tc_f64(Plan* p, int t, const float* Z32, int z32_pitch, const double* dc, double* Zhat, int n_img,
                  int zrows, cudaStream_t st) {
  return wiener_tc_t<double>(p, t, Z32, z32_pitch, dc, Zhat, n_img, zrows, st);
}

}  // namespace fepll
