// Kernel (c): Wiener estimates on the FP64 tensor cores (DMMA).
//
// Restates pkg/src/fepll/gmm.py:352-359 for every patch of a leaf bucket
// (the grouping of pkg/src/fepll/solver.py:233-241):
//     C    = (Z U_k) * (gamma - gamma_tail)        64 x r
//     Zhat = C U_k^T + gamma_tail Z                64 x P
// and writes Zhat + dc (the reprojection input of pkg/src/fepll/patches.py:
// 198-222, `vals = est + dc`, rounded once here instead of in kernel (d)),
// in FP64 — the estimates become the next iteration's image, whose tree
// decisions must stay the FP64 reference's, so no reduced precision here.
//
// A CTA (MT/8 warps) walks a contiguous range of MT-patch tiles in leaf order:
// U_k is staged in smem once per leaf, the FP64 patch rows (kernel (a)
// output, 512 B each) arrive by cp.async into a double buffer while the
// previous tile computes.  Both products run as mma.sync m16n8k8 f64
// (37.2 TFLOP/s FP64 peak measured on B200 for every f64 shape,
// tools/dmma_bench.cu; the k8 shape halves the B-fragment loads per FLOP of
// m8n8k4): warp w owns rows 16w..16w+15 of the tile.
#include <type_traits>

#include "route.cuh"

namespace fepll {

namespace wn {

// debug timeline (fepll_debug_wiener_trace): [CTA][64 tiles][8] clock64
__device__ uint64_t* g_trace = nullptr;
// (callers test a trace flag read once per CTA: a global load of g_trace per
// stamp stalled every tile behind its barrier)
__device__ __forceinline__ void wstamp(int i, int slot) {
  if (i < 64 && threadIdx.x == 0 && blockIdx.x < 148) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    g_trace[((size_t)blockIdx.x * 64 + i) * 8 + slot] = t;
  }
}

constexpr int kMaxP = 128;
constexpr int kMaxR = 64;
constexpr int kMaxRows = 128;

// tile rows MT: 64 (8 warps) for small buckets, 128 (16 warps, twice the
// independent DMMA chains per SM) when the buckets are large
struct Head {
  int32_t tpre[kMaxLevelNodes + 1];
  uint64_t scan_tmp[256];
  int32_t leaf_cr[kMaxLevelNodes];  // component | rank << 16, bucket count and offset,
  int32_t leaf_cnt[kMaxLevelNodes]; // gamma_tail at this iteration: every per-tile
  double leaf_gt[kMaxLevelNodes];   // constant from smem (no global round trip per tile)
  int64_t leaf_off[kMaxLevelNodes];
  int32_t rows[8][kMaxRows];        // patch-index ring (2 x stages slots)
  int32_t t_begin, t_end;
};

// D(16x8) += A(16x8) B(8x8); lane (g = lane/4, t = lane%4) holds
// a = {A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4]}, b = {B[t][g], B[t+4][g]},
// d = {D[g][2t], D[g][2t+1], D[g+8][2t], D[g+8][2t+1]}
// D(8x8) += A(8x4) B(4x8): lane (g, t) holds a = A[g][t], b = B[t][g],
// d = {D[g][2t], D[g][2t+1]}.  Not volatile: ptxas may interleave the
// independent accumulators (each m16n8k8 is four of these).
__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma16(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
// src_bytes 0: the destination is zero-filled, nothing is read
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8z(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Row strides (in doubles) are 4 mod 16: a lane (g, t) fragment load of
// row g, col t (A side) or of row t, col g (phase 1's B side, Us[p][j]) and
// phase 2's B side read straight from Us (row 8n + g, col k + t) all hit 16
// distinct 8-byte banks per half-warp — one basis copy serves both phases.
struct Geo {
  int P, Pn;     // P, P rounded up to 8 (phase-1 K, phase-2 N)
  int zld;       // Zs [MT][zld], columns P..Pn-1 zero
  int R8;        // rank rounded up to 8
  int uld;       // Us [Pn][uld]  (phase-1 B: k = p, n = j; phase-2 B: k = j, n = p)
  int add_dc;    // 1: write est + dc (default), 0: the bare estimates (plan option wiener_add_dc)
  int zld32;     // row stride (floats) of the FP32-row variant: 4 mod 32, conflict-free fragment loads
  int R8e;       // R8 rounded up to 16: basis / shrink columns staged (zero past the rank)
};

// NT2: phase-2 n-tiles (P/8 rounded up): 8 for P=64, 13 for P=100.
// MT rows per tile, NS row buffers (NS - 1 tiles of rows in flight).
// One warp's 16 rows, NT1 = rank n-tiles of 8 (compile time: predicated-off
// DMMAs would still occupy the pipe):
//   phase 1: C = (Z . U) * shrink, accumulators in registers;
//   phase 2: acc2 = C . U^T, its A fragments taken from phase 1's
//            accumulators by quad shuffles (no shared-memory round trip).
// za / zb: this lane's A rows (g, g + 8) at column t.  step(s), s = 0 ..
// NT2-1, runs before phase-1 k-step s: the caller issues the next tile's row
// copies there, so their issue shares the SM with the DMMAs instead of
// preceding them.
// RW = 16: the warp's rows g and g + 8 (two DMMAs per B fragment); RW = 8:
// row g only (half the accumulators and registers, twice the warps per SM)
template <int NT2, int NT1, int RW, class ZT, class Step>
__device__ __forceinline__ void wiener_rows(const ZT* za, const ZT* zb, double da, double db,
                                            const double* Us, int uld, const double* sh, int t4,
                                            int g4, Step&& step, double (&acc2)[NT2][4]) {
  double acc[NT1][4];
#pragma unroll
  for (int n = 0; n < NT1; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < NT2 * 8; k0 += 8) {  // NT2 * 8 == Pn
    step(k0 / 8);
    // z = window - dc, the extraction's FP64 subtraction (da = db = 0 when
    // the rows are already z: x - 0 is x for every x, signed zeros included)
    const double a0 = (double)za[k0] - da, a2 = (double)za[k0 + 4] - da;
    const double a1 = RW == 16 ? (double)zb[k0] - db : 0.0, a3 = RW == 16 ? (double)zb[k0 + 4] - db : 0.0;
    const double* u0 = Us + (k0 + t4) * uld + g4;
    const double* u1 = u0 + 4 * uld;
    double b0[NT1], b1[NT1];
#pragma unroll
    for (int n = 0; n < NT1; ++n) {
      b0[n] = u0[n * 8];
      b1[n] = u1[n * 8];
    }
    if constexpr (RW == 16) {
      // one m16n8k8 per n-tile: bitwise the two m8n8k4 steps per row half
      // below (DMMA accumulates k in order, tools/dmma_order_probe.cu) at a
      // quarter of the instructions
      const double af[4] = {a0, a1, a2, a3};
#pragma unroll
      for (int n = 0; n < NT1; ++n) {
        const double bf[2] = {b0[n], b1[n]};
        dmma16(acc[n], af, bf);
      }
    } else {
      // m8n8k4 steps, consecutive DMMAs on different accumulators (k 0-3
      // for every n, then k 4-7)
#pragma unroll
      for (int n = 0; n < NT1; ++n) dmma8(acc[n][0], acc[n][1], a0, b0[n]);
#pragma unroll
      for (int n = 0; n < NT1; ++n) dmma8(acc[n][0], acc[n][1], a2, b1[n]);
    }
  }
  // C = acc * shrink: lane (g, t) holds C[g][8n + 2t + e] (acc[n][e]) and
  // C[g + 8][8n + 2t + e] (acc[n][2 + e])
#pragma unroll
  for (int n = 0; n < NT1; ++n) {
    const int col = n * 8 + 2 * t4;
    acc[n][0] *= sh[col];
    acc[n][1] *= sh[col + 1];
    if (RW == 16) {
      acc[n][2] *= sh[col];
      acc[n][3] *= sh[col + 1];
    }
  }
#pragma unroll
  for (int n = 0; n < NT2; ++n) acc2[n][0] = acc2[n][1] = acc2[n][2] = acc2[n][3] = 0.0;
  // phase-2 A fragment of k-tile kb: a = {C[g][8kb + t], C[g+8][8kb + t],
  // C[g][8kb + 4 + t], C[g+8][8kb + 4 + t]}; column 8kb + c sits in lane
  // (g, c / 2), element c % 2
  const int q0 = (g4 << 2) | (t4 >> 1), q1 = q0 + 2;
  const bool odd = t4 & 1;
#pragma unroll
  for (int kb = 0; kb < NT1; ++kb) {
    double a[4];
    {
      // the source lane sends the element the receiver's parity needs
      const double e0 = __shfl_sync(0xffffffffu, acc[kb][0], q0), e1 = __shfl_sync(0xffffffffu, acc[kb][1], q0);
      const double h0 = __shfl_sync(0xffffffffu, acc[kb][0], q1), h1 = __shfl_sync(0xffffffffu, acc[kb][1], q1);
      a[0] = odd ? e1 : e0;
      a[2] = odd ? h1 : h0;
      if (RW == 16) {
        const double f0 = __shfl_sync(0xffffffffu, acc[kb][2], q0), f1 = __shfl_sync(0xffffffffu, acc[kb][3], q0);
        const double j0 = __shfl_sync(0xffffffffu, acc[kb][2], q1), j1 = __shfl_sync(0xffffffffu, acc[kb][3], q1);
        a[1] = odd ? f1 : f0;
        a[3] = odd ? j1 : j0;
      } else {
        a[1] = a[3] = 0.0;
      }
    }
    const double* u0 = Us + g4 * uld + 8 * kb + t4;  // U[8n + g][k + t] = U^T[k][n]
    double b0[NT2], b1[NT2];
#pragma unroll
    for (int n = 0; n < NT2; ++n) {
      b0[n] = u0[n * 8 * uld];
      b1[n] = u0[n * 8 * uld + 4];
    }
    if constexpr (RW == 16) {
#pragma unroll
      for (int n = 0; n < NT2; ++n) {
        const double bf[2] = {b0[n], b1[n]};
        dmma16(acc2[n], a, bf);
      }
    } else {
#pragma unroll
      for (int n = 0; n < NT2; ++n) dmma8(acc2[n][0], acc2[n][1], a[0], b0[n]);
#pragma unroll
      for (int n = 0; n < NT2; ++n) dmma8(acc2[n][0], acc2[n][1], a[2], b1[n]);
    }
  }
}

// PAIR (split) form: warps 2q, 2q + 1 share rows 16q .. 16q + 15 and issue
// m16n8k8 DMMAs (16 rows x 8 columns x 8 k each, bitwise the m8n8k4 pairs:
// tools/dmma_order_probe.cu) — a quarter of the DMMA instructions and half
// the basis fragment loads per flop of the 8-row warps, at the same 16
// warps per SM: warp half hf takes rank tiles [hf NH, (hf+1) NH) in phase 1
// and column tiles [hf NT2/2, (hf+1) NT2/2) in phase 2, C crossing between
// the two warps through shared memory (Cs, 16 x uld per pair).
template <int NT2, int NH, class ZT, class Step>
__device__ __forceinline__ void wiener_rows_pair(const ZT* za, const ZT* zb, const double* Us, int uld,
                                                 const double* sh, int t4, int g4, int hf, double* Cs,
                                                 int bar_id, Step&& step, double (&acc2)[NT2 / 2][4]) {
  double acc[NH][4];
#pragma unroll
  for (int n = 0; n < NH; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0;
  const int c0 = hf * NH * 8;  // this warp's first rank column
#pragma unroll
  for (int k0 = 0; k0 < NT2 * 8; k0 += 8) {  // NT2 * 8 == Pn
    step(k0 / 8);
    const double af[4] = {(double)za[k0], (double)zb[k0], (double)za[k0 + 4], (double)zb[k0 + 4]};
    const double* u0 = Us + (k0 + t4) * uld + g4 + c0;
    const double* u1 = u0 + 4 * uld;
#pragma unroll
    for (int n = 0; n < NH; ++n) {
      const double bf[2] = {u0[n * 8], u1[n * 8]};
      dmma16(acc[n], af, bf);
    }
  }
  // C = acc * shrink (rows g, g + 8; columns c0 + 8n + 2t, + 1)
#pragma unroll
  for (int n = 0; n < NH; ++n) {
    const int col = c0 + n * 8 + 2 * t4;
    Cs[g4 * uld + col] = acc[n][0] * sh[col];
    Cs[g4 * uld + col + 1] = acc[n][1] * sh[col + 1];
    Cs[(g4 + 8) * uld + col] = acc[n][2] * sh[col];
    Cs[(g4 + 8) * uld + col + 1] = acc[n][3] * sh[col + 1];
  }
  asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
#pragma unroll
  for (int n = 0; n < NT2 / 2; ++n) acc2[n][0] = acc2[n][1] = acc2[n][2] = acc2[n][3] = 0.0;
  const int n0 = hf * (NT2 / 2);
#pragma unroll
  for (int kb = 0; kb < 2 * NH; ++kb) {
    const double af[4] = {Cs[g4 * uld + 8 * kb + t4], Cs[(g4 + 8) * uld + 8 * kb + t4],
                          Cs[g4 * uld + 8 * kb + 4 + t4], Cs[(g4 + 8) * uld + 8 * kb + 4 + t4]};
    const double* u0 = Us + g4 * uld + 8 * kb + t4;  // U[8n + g][k + t] = U^T[k][n]
#pragma unroll
    for (int n = 0; n < NT2 / 2; ++n) {
      const double bf[2] = {u0[(n0 + n) * 8 * uld], u0[(n0 + n) * 8 * uld + 4]};
      dmma16(acc2[n], af, bf);
    }
  }
}

// XW: the rows are 8 x 8 windows of the image x (P = 64 only) instead of the
// extracted Z64 rows; z = window - dc is formed at the fragment loads, so the
// extraction need not write (and this kernel not read) the 512-byte Z64 rows
// (off by default: slower, see plan option wiener_xw).
// ZT: element type of the patch rows in and the estimate rows out (double;
// float for the FP32-state mode — rows converted exactly to FP64 at the
// fragment loads, the FP64 result rounded once to FP32 at the store)
template <int NT2, int MT, int NS, int RW, bool XW, class ZT = double, bool PAIR = false>
__global__ void __launch_bounds__(PAIR ? MT / 16 * 64 : MT / RW * 32, (RW == 8 || PAIR) ? 2 : 1)
wiener_dmma_kernel(PlanView pv, int t, const int32_t* __restrict__ leaf_nodes, int n_leaf_nodes,
                   const int32_t* __restrict__ cnt, const int64_t* __restrict__ off,
                   const int32_t* __restrict__ leafseg, const ZT* __restrict__ Z64, int zin_pitch,
                   const double* __restrict__ dc, ZT* __restrict__ Zhat, int n_img, int zrows,
                   const double* __restrict__ x, const int32_t* __restrict__ anchors, int H, int W,
                   Geo geo) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int kRows = MT;
  constexpr int kThreads = PAIR ? MT / 16 * 64 : MT / RW * 32;  // one warp (pair) per RW (16) rows
  static_assert(!PAIR || (RW == 16 && !XW && NT2 % 2 == 0), "PAIR: 16-row warp pairs, even column tiles");
  Head& h = *reinterpret_cast<Head*>(smem);
  constexpr int kRing = 2 * NS;      // index ring slots
  // tiles of indices fetched ahead of their rows' issue (XW: one more, for
  // the anchors fetched between the index and the window copies)
  constexpr int kLead = XW ? 2 * NS - 1 : 2 * NS - 2;
  static_assert(!XW || (NS == 2 && NT2 == 8), "XW: the P = 64 two-stage pipeline");
  static_assert(!XW || sizeof(ZT) == 8, "XW reads FP64 windows");
  constexpr int kEl = 16 / (int)sizeof(ZT);   // row elements per 16-byte copy
  const int zld = sizeof(ZT) == 8 ? geo.zld : geo.zld32;
  ZT* Zs0 = reinterpret_cast<ZT*>(smem + ((sizeof(Head) + 127) & ~size_t(127)));
  double* Us = reinterpret_cast<double*>(
      reinterpret_cast<uint8_t*>(Zs0) + ((NS * kRows * zld * sizeof(ZT) + 15) & ~size_t(15)));  // [Pn][uld] (p, j)
  double* sh = Us + geo.Pn * geo.uld;          // [R8e]
  double* dcs = sh + geo.R8e;                  // [NS][MT] dc of the buffered rows
  int2* anc = reinterpret_cast<int2*>(dcs + NS * kRows);  // XW: [4][MT] anchors of the rows
  double* Cs = reinterpret_cast<double*>(anc + 4 * kRows);  // PAIR: [MT][uld] C of the tile
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = geo.P;
  const bool trace_on = g_trace != nullptr;
  // K padding columns of the row buffers stay zero (cp.async fills [0, P))
  for (int e = tid; e < NS * kRows * (geo.Pn - P); e += kThreads) {
    const int w = geo.Pn - P, i = e / w;  // row i of the adjacent buffers
    Zs0[i * zld + P + (e - i * w)] = (ZT)0;
  }
  for (int k = tid; k < n_leaf_nodes; k += kThreads) {
    const int v = leaf_nodes[k];
    const int comp = pv.leaf_index[v];
    h.leaf_cr[k] = comp | (pv.model_rank[comp] << 16);
    h.leaf_gt[k] = pv.model_gamma_tail[(int64_t)t * pv.K + comp];
    h.leaf_cnt[k] = cnt[v];
    h.leaf_off[k] = off[v];
    h.tpre[k] = (cnt[v] + kRows - 1) / kRows;
  }
  __syncthreads();
  const int tiles = block_exscan(h.tpre, n_leaf_nodes, h.scan_tmp);
  if (tid == 0) {
    h.tpre[n_leaf_nodes] = tiles;
    h.t_begin = (int)(((int64_t)tiles * blockIdx.x) / gridDim.x);
    h.t_end = (int)(((int64_t)tiles * (blockIdx.x + 1)) / gridDim.x);
  }
  __syncthreads();
  const int t_begin = h.t_begin, t_end = h.t_end;
  if (t_begin >= t_end) return;

  // Pipeline (all cp.async): the rows of tile j land in buffer j % NS,
  // issued NS - 1 tiles ahead of its compute; its patch indices land in ring
  // slot j % kRing another NS - 1 tiles earlier — no global round trip on
  // the compute path, NS - 1 tiles of random 8P-byte row reads in flight.
  int fli = prefix_find(h.tpre, n_leaf_nodes, t_begin);  // leaf of the next index fetch
  int cli = fli;                                         // leaf of the computed tile
  auto fetch_rows = [&](int j) {
    if (j < t_end && tid < kRows) {
      while (fli + 1 < n_leaf_nodes && h.tpre[fli + 1] <= j) ++fli;  // tiles ascend
      const int li = fli;
      const int first = (j - h.tpre[li]) * kRows;
      int32_t* dst = &h.rows[(j - t_begin) % kRing][tid];
      if (tid < h.leaf_cnt[li] - first)
        cp_async4(dst, leafseg + h.leaf_off[li] + first + tid);
      else
        *dst = -1;
    }
  };
  // consecutive threads take consecutive 16-byte chunks of a row (P even),
  // so each instruction reads whole lines of one or two rows; slice s of a
  // tile's copy is e in [s kThreads, (s + 1) kThreads)
  const int C = P / kEl;
  const int n_slices = (kRows * C + kThreads - 1) / kThreads;
  constexpr int kWarps = kThreads / 32;
  constexpr bool kInterleave = NT2 == 8;  // P = 64 layout below: 16 slices, 8 k-steps
  auto fetch_anc = [&](int j) {  // XW: anchors of tile j's rows (indices landed)
    if (XW && j < t_end && tid < kRows) {
      const int g = h.rows[(j - t_begin) % kRing][tid];
      if (g >= 0) cp_async8(&anc[((j - t_begin) & 3) * kRows + tid], anchors + 2 * (g % n_img));
    }
  };
  // XW: thread chunk c (16 bytes = window columns 2(c%4), +1 of window row
  // c/4) of row i of tile j; odd anchor columns are 8-byte aligned only
  auto copy_window_chunk = [&](int j, int i, int c, int g, double* d) {
    const int2 a = anc[((j - t_begin) & 3) * kRows + i];
    const int b = g / n_img;
    const double* src = x + ((int64_t)b * H + a.x + (c >> 2)) * W + a.y + 2 * (c & 3);
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      cp_async16(d, src);
    } else {
      cp_async8(d, src);
      cp_async8(d + 1, src + 1);
    }
  };
  auto fetch_z_slices = [&](int j, int s0, int s1) {
    if (j >= t_end) return;
    const int32_t* rows = h.rows[(j - t_begin) % kRing];
    ZT* Zs = Zs0 + ((j - t_begin) % NS) * kRows * zld;
    double* dcb = dcs + ((j - t_begin) % NS) * kRows;
    for (int e = tid + s0 * kThreads; e < min(s1 * kThreads, kRows * C); e += kThreads) {
      const int i = e / C, c = e - i * C;
      const int g = rows[i];
      ZT* d = Zs + i * zld + kEl * c;
      if (g >= 0) {
        if constexpr (XW)
          copy_window_chunk(j, i, c, g, d);
        else
          cp_async16(d, Z64 + (int64_t)g * zin_pitch + kEl * c);
        if (c == 0) cp_async8(dcb + i, dc + g);
      } else {
#pragma unroll
        for (int q = 0; q < kEl; ++q) d[q] = (ZT)0;
      }
    }
  };

  int cur_leaf = -1;
  for (int j = 0; j < kLead; ++j) fetch_rows(t_begin + j);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  if (XW) {
    fetch_anc(t_begin);
    fetch_anc(t_begin + 1);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  for (int j = 0; j < NS - 1; ++j) {
    fetch_z_slices(t_begin + j, 0, n_slices);
    cp_async_commit();
  }
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int i = tile - t_begin;
    const int slot = i % kRing;
    while (cli + 1 < n_leaf_nodes && h.tpre[cli + 1] <= tile) ++cli;  // tiles ascend
    const int li = cli;
    const int comp = h.leaf_cr[li] & 0xFFFF;
    const int r = h.leaf_cr[li] >> 16;
    if (trace_on) wstamp(i, 0);
    bulk_wait_read();  // the previous tile's row stores have left its buffer
    cp_async_wait_group<NS - 2>();
    __syncthreads();  // this tile's rows landed; the buffer refilled next is free
    if (trace_on) wstamp(i, 1);
    fetch_rows(tile + kLead);  // committed with the row copies below (one group per tile)
    fetch_anc(tile + 2);       // XW: its indices landed with the last group
    if (comp != cur_leaf) {
      const double* U = pv.model_basis + pv.model_off64[comp];
      for (int e = tid; e < geo.Pn * geo.R8e; e += kThreads) {
        const int p = e / geo.R8e, j = e - p * geo.R8e;
        const double u = (p < P && j < r) ? U[(int64_t)p * r + j] : 0.0;
        Us[p * geo.uld + j] = u;
      }
      const double* shrink = pv.model_shrink + (int64_t)t * pv.model_cols_total + pv.model_col_off[comp];
      for (int j = tid; j < geo.R8e; j += kThreads) sh[j] = j < r ? shrink[j] : 0.0;
      cur_leaf = comp;
      __syncthreads();
    }
    if (trace_on) wstamp(i, 2);
    const ZT* Zs = Zs0 + (i % NS) * kRows * zld;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int m0 = PAIR ? (warp >> 1) * 16 : warp * RW;
    const ZT* za = Zs + (m0 + g4) * zld + t4;       // rows g (, g+8) of the warp
    const ZT* zb = za + 8 * zld;
    // ---- phase 1: C[m0..m0+15][0..R8) = (Z . U) * shrink, with the
    // leaf's n-tile count as a compile-time constant (predicated-off DMMAs
    // would still occupy the pipe)
    // The next tile's row copies.  P = 64: thread (w, l) copies chunk l of
    // rows w + kWarps s, s = 0..15, two per phase-1 k-step, with
    // the patch indices read up front (an index load feeding each copy would
    // stall the warp's in-order DMMA issue behind it); other shapes issue
    // the whole copy here.
    const int jn = tile + NS - 1;
    const bool inter = kInterleave && P == 64 && jn < t_end;
    constexpr int kRowsPerThread = kRows / kWarps;  // == RW: RW / 8 rows per k-step
    int gsl[kRowsPerThread];
    int2 asl[XW ? kRowsPerThread : 1];
    ZT* zn = Zs0 + ((jn - t_begin) % NS) * kRows * zld + kEl * lane;
    double* dcn = dcs + ((jn - t_begin) % NS) * kRows;
    if (inter) {
      const int32_t* rn = h.rows[(jn - t_begin) % kRing];
#pragma unroll
      for (int q = 0; q < kRowsPerThread; ++q) gsl[q] = rn[warp + kWarps * q];
      if (XW) {
        const int2* an = anc + ((jn - t_begin) & 3) * kRows;
#pragma unroll
        for (int q = 0; q < kRowsPerThread; ++q) asl[XW ? q : 0] = an[warp + kWarps * q];
      }
    } else {
      fetch_z_slices(jn, 0, n_slices);
    }
    // this lane's 16-byte chunk of every Z64 row (rows past the bucket: zero-filled)
    const ZT* zsrc = Z64 + kEl * lane;
    auto zstep = [&](int st) {
      if (!inter) return;
#pragma unroll
      for (int q = st * (kRowsPerThread / 8); q < (st + 1) * (kRowsPerThread / 8); ++q) {
        ZT* d = zn + (warp + kWarps * q) * zld;
        if (kEl * lane >= 64) continue;  // FP32 rows: 16 lanes cover the 256-byte row
        if constexpr (!XW) {
          const int g = gsl[q];
          const bool ok = g >= 0;
          cp_async16z(d, ok ? zsrc + (int64_t)g * zin_pitch : zsrc, ok ? 16u : 0u);
          if (lane == 0) cp_async8z(dcn + warp + kWarps * q, ok ? dc + g : dc, ok ? 8u : 0u);
          continue;
        }
        if (gsl[q] >= 0) {
          if constexpr (XW) {
            const int2 a = asl[XW ? q : 0];
            const int b = gsl[q] / n_img;
            const double* src = x + ((int64_t)b * H + a.x + (lane >> 2)) * W + a.y + 2 * (lane & 3);
            if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
              cp_async16(d, src);
            } else {
              cp_async8(d, src);
              cp_async8(d + 1, src + 1);
            }
          } else {
            cp_async16(d, Z64 + (int64_t)gsl[q] * zin_pitch + kEl * lane);
          }
          if (lane == 0) cp_async8(dcn + warp + kWarps * q, dc + gsl[q]);
        } else {
#pragma unroll
          for (int e2 = 0; e2 < kEl; ++e2) d[e2] = (ZT)0;
        }
      }
    };
    constexpr int kNA = PAIR ? NT2 / 2 : NT2;  // column tiles of this warp
    double acc[kNA][4];
    const double* dcc = dcs + (i % NS) * kRows;  // dc of this tile's rows
    const double da = XW ? dcc[m0 + g4] : 0.0;
    const double db = XW && RW == 16 ? dcc[m0 + g4 + 8] : 0.0;
    const int hf = warp & 1;
    const int bar_id = 1 + (warp >> 1);
    double* Cp = Cs + m0 * geo.uld;
    if constexpr (PAIR) {
      // rank tiles per half: ceil(r / 16) (zero basis columns up to R8e)
      switch ((r + 15) / 16) {
        case 1: wiener_rows_pair<NT2, 1>(za, zb, Us, geo.uld, sh, t4, g4, hf, Cp, bar_id, zstep,
                                         acc); break;
        case 2: wiener_rows_pair<NT2, 2>(za, zb, Us, geo.uld, sh, t4, g4, hf, Cp, bar_id, zstep,
                                         acc); break;
        case 3: wiener_rows_pair<NT2, 3>(za, zb, Us, geo.uld, sh, t4, g4, hf, Cp, bar_id, zstep,
                                         acc); break;
        default: wiener_rows_pair<NT2, 4>(za, zb, Us, geo.uld, sh, t4, g4, hf, Cp, bar_id, zstep,
                                          acc); break;
      }
    } else
    switch ((r + 7) / 8) {
      case 1: wiener_rows<NT2, 1, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      case 2: wiener_rows<NT2, 2, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      case 3: wiener_rows<NT2, 3, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      case 4: wiener_rows<NT2, 4, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      case 5: wiener_rows<NT2, 5, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      case 6: wiener_rows<NT2, 6, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      case 7: wiener_rows<NT2, 7, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
      default: wiener_rows<NT2, 8, RW>(za, zb, da, db, Us, geo.uld, sh, t4, g4, zstep, acc); break;
    }
    cp_async_commit();
    if (trace_on) wstamp(i, 3);
    {
      if (trace_on) wstamp(i, 4);
      const double gt = h.leaf_gt[li];
      // Zhat + dc = (acc + gamma_tail z) + dc, written over this warp's own
      // rows of Zs (each element read and written by the same lane)...
      ZT* zw = const_cast<ZT*>(Zs);
      const double* dct = dcs + (i % NS) * kRows;
#pragma unroll
      for (int half = 0; half < RW / 8; ++half) {
        ZT* zr = zw + (m0 + g4 + 8 * half) * zld;
        const double d = dct[m0 + g4 + 8 * half];
        const double dz = XW ? d : 0.0;  // XW rows hold the window: z = w - dc
#pragma unroll
        for (int n = 0; n < kNA; ++n) {
          const int col = ((PAIR ? hf * kNA : 0) + n) * 8 + 2 * t4;
          if (col < P) {
            const double e0 = acc[n][2 * half] + gt * ((double)zr[col] - dz);
            const double e1 = acc[n][2 * half + 1] + gt * ((double)zr[col + 1] - dz);
            zr[col] = (ZT)(geo.add_dc ? __dadd_rn(e0, d) : e0);
            zr[col + 1] = (ZT)(geo.add_dc ? __dadd_rn(e1, d) : e1);
          }
        }
      }
      // ... then each of the warp's 16 rows leaves as one TMA bulk store
      // (smem -> global, 8P bytes); the buffer is reused only after the
      // stores have read it (wait_group.read before the next tile's barrier;
      // coalesced 16-byte stores from the same rows measured slower)
      fence_proxy_async_smem();
      __syncwarp();
      if (PAIR) asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // both column halves written
      if (lane < RW && (!PAIR || hf == 0)) {
        const int gidx = h.rows[slot][m0 + lane];
        if (gidx >= 0) {
          const int64_t orow =  // padded image pitch (no division when dense)
              zrows == n_img ? (int64_t)gidx : (int64_t)(gidx / n_img) * zrows + gidx % n_img;
          bulk_s2g(Zhat + orow * P, zw + (m0 + lane) * zld, P * (uint32_t)sizeof(ZT));
        }
        bulk_commit();
      }
      if (trace_on) wstamp(i, 5);
    }
  }
  bulk_wait_all();  // the last rows' stores are complete before the kernel ends
}


// ---------------------------------------------------------------------------
// Warp-specialised form (plan option wiener_ws; P = 64, FP64 rows): one CTA
// per SM, 12 compute warps (8 rows each of a 96-row tile: the same DMMA
// sequence per element as wiener_dmma_kernel<8, 64, 2, 8>, bitwise the same
// estimates) and 2 loader warps that run two tiles ahead (patch indices one
// tile further) through a three-stage ring of row buffers guarded by
// mbarriers.  A compute warp never meets a CTA barrier between tiles: it
// waits for its tile's rows, runs both products and the epilogue on its own
// 8 rows, hands them to the TMA as bulk stores and moves on; the stage goes
// back to the loaders once every warp's stores have read it.  The FP64 pipe
// keeps the other warps' DMMAs while one warp is in its epilogue (the
// two-CTA kernel holds ~64 % of the pipe: all 8 warps of a CTA reach their
// barrier, epilogue and stores together).
namespace ws {
constexpr int kCW = 12;               // compute warps
constexpr int kLW = 2;                // loader warps
constexpr int kThreads = 32 * (kCW + kLW);
constexpr int kMT = 8 * kCW;          // rows per tile
constexpr int kNS = 3;                // row stages
constexpr int kRing = kNS + 3;        // index ring slots

struct Head {
  int32_t tpre[kMaxLevelNodes + 1];
  uint64_t scan_tmp[256];
  int32_t leaf_cr[kMaxLevelNodes];
  int32_t leaf_cnt[kMaxLevelNodes];
  double leaf_gt[kMaxLevelNodes];
  int64_t leaf_off[kMaxLevelNodes];
  int32_t rows[kRing][kMT];
  uint64_t full[kNS], empty[kNS];
  int32_t t_begin, t_end;
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
wiener_ws_kernel(PlanView pv, int t, const int32_t* __restrict__ leaf_nodes, int n_leaf_nodes,
                 const int32_t* __restrict__ cnt, const int64_t* __restrict__ off,
                 const int32_t* __restrict__ leafseg, const double* __restrict__ Z64,
                 const double* __restrict__ dc, double* __restrict__ Zhat, int n_img, int zrows, Geo geo) {
  extern __shared__ __align__(16) uint8_t smem[];
  Head& h = *reinterpret_cast<Head*>(smem);
  constexpr int P = 64;
  const int zld = geo.zld;
  double* Zs0 = reinterpret_cast<double*>(smem + ((sizeof(Head) + 127) & ~size_t(127)));  // [kNS][kMT][zld]
  double* Us = Zs0 + (size_t)kNS * kMT * zld;  // [64][uld]
  double* sh = Us + 64 * geo.uld;              // [R8e]
  double* dcs = sh + geo.R8e;                  // [kNS][kMT]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&h.full[i], 32 * kLW);
      mbar_init(&h.empty[i], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = tid; k < n_leaf_nodes; k += kThreads) {
    const int v = leaf_nodes[k];
    const int comp = pv.leaf_index[v];
    h.leaf_cr[k] = comp | (pv.model_rank[comp] << 16);
    h.leaf_gt[k] = pv.model_gamma_tail[(int64_t)t * pv.K + comp];
    h.leaf_cnt[k] = cnt[v];
    h.leaf_off[k] = off[v];
    h.tpre[k] = (cnt[v] + kMT - 1) / kMT;
  }
  __syncthreads();
  const int tiles = block_exscan(h.tpre, n_leaf_nodes, h.scan_tmp);
  if (tid == 0) {
    h.tpre[n_leaf_nodes] = tiles;
    h.t_begin = (int)(((int64_t)tiles * blockIdx.x) / gridDim.x);
    h.t_end = (int)(((int64_t)tiles * (blockIdx.x + 1)) / gridDim.x);
  }
  __syncthreads();
  const int t_begin = h.t_begin, t_end = h.t_end;
  const int ntile = t_end - t_begin;

  if (warp >= kCW) {
    // ------------------------------------------------------------ loaders
    const int lt = tid - 32 * kCW;  // 0 .. 63
    int fli = prefix_find(h.tpre, n_leaf_nodes, t_begin);
    auto issue_idx = [&](int j) {  // tile t_begin + j: its patch indices into ring slot j % kRing
      if (j < ntile) {
        const int tile = t_begin + j;
        while (fli + 1 < n_leaf_nodes && h.tpre[fli + 1] <= tile) ++fli;
        const int first = (tile - h.tpre[fli]) * kMT;
        for (int r = lt; r < kMT; r += 32 * kLW) {
          int32_t* dst = &h.rows[j % kRing][r];
          if (r < h.leaf_cnt[fli] - first) cp_async4(dst, leafseg + h.leaf_off[fli] + first + r);
          else *dst = -1;
        }
      }
    };
    issue_idx(0);
    cp_async_commit();
    issue_idx(1);
    cp_async_commit();
    issue_idx(2);
    cp_async_commit();
    for (int j = 0; j < ntile; ++j) {
      const int st = j % kNS;
      if (j >= kNS) mbar_wait(&h.empty[st], ((j / kNS) - 1) & 1);
      cp_async_wait_group<2>();  // idx(j) landed (this thread's copies; the barrier below covers the others)
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kLW) : "memory");
      const int32_t* rows = h.rows[j % kRing];
      double* Zs = Zs0 + (size_t)st * kMT * zld;
      // 32 chunks of 16 bytes per row: a warp instruction copies one whole row
      for (int e = lt; e < kMT * 32; e += 32 * kLW) {
        const int i = e >> 5, c = e & 31;
        const int g = rows[i];
        const bool ok = g >= 0;
        cp_async16z(Zs + i * zld + 2 * c, ok ? Z64 + (int64_t)g * P + 2 * c : Z64, ok ? 16u : 0u);
        if (c == 0) cp_async8z(dcs + st * kMT + i, ok ? dc + g : dc, ok ? 8u : 0u);
      }
      issue_idx(j + 3);
      cp_async_commit();
      cp_async_mbar_arrive(&h.full[st]);
    }
    cp_async_wait_all();
    return;
  }

  // -------------------------------------------------------------- compute
  const int g4 = lane >> 2, t4 = lane & 3;
  const int m0 = warp * 8;
  int cli = prefix_find(h.tpre, n_leaf_nodes, t_begin);
  int cur_leaf = -1;
  for (int j = 0; j < ntile; ++j) {
    const int tile = t_begin + j;
    const int st = j % kNS;
    while (cli + 1 < n_leaf_nodes && h.tpre[cli + 1] <= tile) ++cli;
    const int li = cli;
    const int comp = h.leaf_cr[li] & 0xFFFF;
    const int r = h.leaf_cr[li] >> 16;
    if (comp != cur_leaf) {
      // every compute warp is done with the previous leaf's basis
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kCW) : "memory");
      const double* U = pv.model_basis + pv.model_off64[comp];
      for (int e = tid; e < 64 * geo.R8e; e += 32 * kCW) {
        const int p = e / geo.R8e, q = e - p * geo.R8e;
        Us[p * geo.uld + q] = q < r ? U[(int64_t)p * r + q] : 0.0;
      }
      const double* shrink = pv.model_shrink + (int64_t)t * pv.model_cols_total + pv.model_col_off[comp];
      for (int q = tid; q < geo.R8e; q += 32 * kCW) sh[q] = q < r ? shrink[q] : 0.0;
      cur_leaf = comp;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kCW) : "memory");
    }
    mbar_wait(&h.full[st], (j / kNS) & 1);
    double* Zs = Zs0 + (size_t)st * kMT * zld;
    const double* za = Zs + (m0 + g4) * zld + t4;
    double acc[8][4];
    auto nostep = [](int) {};
    switch ((r + 7) / 8) {
      case 1: wiener_rows<8, 1, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      case 2: wiener_rows<8, 2, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      case 3: wiener_rows<8, 3, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      case 4: wiener_rows<8, 4, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      case 5: wiener_rows<8, 5, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      case 6: wiener_rows<8, 6, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      case 7: wiener_rows<8, 7, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
      default: wiener_rows<8, 8, 8>(za, za, 0.0, 0.0, Us, geo.uld, sh, t4, g4, nostep, acc); break;
    }
    {
      // Zhat + dc = (acc + gamma_tail z) + dc over this warp's own rows of the stage
      const double gt = h.leaf_gt[li];
      double* zr = Zs + (m0 + g4) * zld;
      const double d = dcs[st * kMT + m0 + g4];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const int col = n * 8 + 2 * t4;
        const double e0 = acc[n][0] + gt * zr[col];
        const double e1 = acc[n][1] + gt * zr[col + 1];
        zr[col] = geo.add_dc ? __dadd_rn(e0, d) : e0;
        zr[col + 1] = geo.add_dc ? __dadd_rn(e1, d) : e1;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane < 8) {
        const int gidx = h.rows[j % kRing][m0 + lane];
        if (gidx >= 0) {
          const int64_t orow = zrows == n_img ? (int64_t)gidx : (int64_t)(gidx / n_img) * zrows + gidx % n_img;
          bulk_s2g(Zhat + orow * P, Zs + (m0 + lane) * zld, P * 8u);
        }
        bulk_commit();
      }
      // the previous tile's stores have read their stage: hand it back
      if (j > 0) {
        bulk_wait_read1();
        __syncwarp();
        if (lane == 0) mbar_arrive(&h.empty[(j - 1) % kNS]);
      }
    }
  }
  bulk_wait_all();
}

}  // namespace ws

}  // namespace wn

static wn::Geo wiener_geo(const Plan* p) {
  const int P = p->v.P;
  wn::Geo geo;
  geo.P = P;
  geo.Pn = (P + 7) / 8 * 8;
  auto ld = [](int n, int rem) { int v = n; while (v % 16 != rem) ++v; return v; };
  geo.zld = ld(geo.Pn, 4);
  geo.zld32 = geo.Pn;
  while (geo.zld32 % 32 != 4) ++geo.zld32;
  geo.R8 = (p->max_model_rank + 7) / 8 * 8;
  geo.R8e = (geo.R8 + 15) / 16 * 16;
  geo.uld = ld(geo.R8, 4);
  geo.add_dc = p->opt.wiener_add_dc;
  return geo;
}

// dynamic shared memory of an (mt rows, ns stages) configuration: head,
// row stages, basis, shrink, dc ring, XW anchors ring
static size_t wiener_smem(const wn::Geo& geo, int mt, int ns, size_t zt_bytes = 8, bool pair = false) {
  const size_t rows = zt_bytes == 8 ? ns * (size_t)mt * geo.zld * 8 : ns * (size_t)mt * geo.zld32 * zt_bytes;
  return ((sizeof(wn::Head) + 127) & ~size_t(127)) + ((rows + 15) & ~size_t(15)) +
         sizeof(double) * ((size_t)geo.Pn * geo.uld + geo.R8e + (size_t)ns * mt) +
         sizeof(int2) * 4 * (size_t)mt + (pair ? sizeof(double) * (size_t)mt * geo.uld : 0);
}

static bool wiener_pair_fits(const wn::Geo& geo) {
  int dev = 0, per_sm_cap = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&per_sm_cap, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess)
    return false;
  return 2 * (wiener_smem(geo, 64, 2) + 1024) <= (size_t)per_sm_cap;
}

// Plan options wiener_pair / wiener_rw: two 64-row CTAs per SM, 8 rows
// per warp (defaults).  Window-source mode (option wiener_xw): measured slower on B200 (64 x 1024^2: extraction
// 3.48 -> 2.06 ms/step without the Z64 writes, but the Wiener kernel 6.8 ->
// 9.3 ms/step gathering 8 x 64-byte window rows per patch instead of one
// 512-byte row), so off by default; it saves the 8P-byte-per-patch Z64
// buffer where HBM capacity matters more.

// the window-source (XW) kernel: P = 64 in the two-CTAs-per-SM, 8-rows-per-
// warp configuration
bool wiener_xw_supported(const Plan* p) {
  return p->opt.wiener_xw && p->v.P == 64 && p->opt.wiener_pair && p->opt.wiener_rw == 8 &&
         p->max_model_rank <= wn::kMaxR && wiener_pair_fits(wiener_geo(p));
}

template <class ZT>
static int wiener_dmma_t(Plan* p, int t, const ZT* Z64, int zin_pitch, const double* dc, ZT* Zhat, int n_img,
                         int zrows, const double* x, const int32_t* anchors, int H, int W, cudaStream_t st) {
  const wn::Geo geo = wiener_geo(p);
  auto smem_for = [&](int mt, int ns) { return wiener_smem(geo, mt, ns, sizeof(ZT)); };
  const bool xw = Z64 == nullptr;
  if constexpr (sizeof(ZT) == 8) {
    // warp-specialised kernel (plan option wiener_ws): P = 64, dense FP64 rows
    const bool ws_on = p->opt.wiener_ws == 1 || (p->opt.wiener_ws == 2 && p->last_n_total >= (1 << 20));
    if (ws_on && !xw && p->v.P == 64 && zin_pitch == 64 && p->max_model_rank <= wn::kMaxR) {
      const size_t smem_ws = ((sizeof(wn::ws::Head) + 127) & ~size_t(127)) +
                             sizeof(double) * ((size_t)wn::ws::kNS * wn::ws::kMT * geo.zld + 64 * (size_t)geo.uld +
                                               geo.R8e + (size_t)wn::ws::kNS * wn::ws::kMT);
      int dev_ws = 0, optin_ws = 0;
      FEPLL_CUDA(cudaGetDevice(&dev_ws));
      FEPLL_CUDA(cudaDeviceGetAttribute(&optin_ws, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev_ws));
      if (smem_ws <= (size_t)optin_ws) {
        FEPLL_CUDA(cudaFuncSetAttribute(wn::ws::wiener_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem_ws));
        wn::ws::wiener_ws_kernel<<<kSMs, wn::ws::kThreads, smem_ws, st>>>(
            p->v, t, p->d_leaf_nodes, p->n_leaf_nodes, p->rs.cnt, p->rs.off, p->rs.leafseg, Z64, dc, Zhat, n_img,
            zrows, geo);
        FEPLL_LAUNCH();
        return kOk;
      }
    }
  }
  FEPLL_REQUIRE(!xw || wiener_xw_supported(p),
                "wiener: the window-source kernel needs P = 64 and two CTAs per SM");
  // 128-row tiles (16 warps) once the average leaf bucket is large enough
  // that the extra padding rows do not matter, and the tile fits in smem
  const int64_t n_total = p->last_n_total;
  int dev = 0, optin = 0;
  FEPLL_CUDA(cudaGetDevice(&dev));
  FEPLL_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t cap = (size_t)optin;
  // 64-row tiles, two CTAs per SM (one CTA's loads, barriers and stores
  // overlap the other's DMMAs) when two fit in shared memory; else 128-row
  // tiles when the buckets are large, else 64-row tiles with deeper staging
  int per_sm_cap = 0;
  FEPLL_CUDA(cudaDeviceGetAttribute(&per_sm_cap, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  const bool pair = p->opt.wiener_pair && 2 * (smem_for(64, 2) + 1024) <= (size_t)per_sm_cap;
  const bool big = !pair && n_total >= (int64_t)1024 * std::max(1, p->n_leaf_nodes) && smem_for(128, 2) <= cap;
  const int mt = big ? 128 : 64;
  const int ns = big || pair ? 2 : (smem_for(64, 4) <= cap ? 4 : 2);
  FEPLL_REQUIRE(smem_for(mt, ns) <= cap, "wiener: tile buffers exceed shared memory");
  const size_t smem = smem_for(mt, ns);
  const int nt2 = geo.Pn / 8;
  const int rw = pair && p->opt.wiener_rw == 8 ? 8 : 16;
  // split warp pairs (m16n8k8, plan option wiener_split): the pair
  // configuration with an even column-tile count and room for the C tiles
  const bool split = pair && !xw && p->opt.wiener_split && nt2 % 2 == 0 && nt2 <= 8 &&
                     2 * (wiener_smem(geo, 64, 2, sizeof(ZT), true) + 1024) <= (size_t)per_sm_cap;
  const size_t smem_launch = split ? wiener_smem(geo, 64, 2, sizeof(ZT), true) : smem;
  const int threads = split ? 256 : mt / rw * 32;
  auto launch = [&](auto kernel) -> int {
    const size_t smem = smem_launch;
    FEPLL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    kernel<<<kSMs * std::max(1, per_sm), threads, smem, st>>>(
        p->v, t, p->d_leaf_nodes, p->n_leaf_nodes, p->rs.cnt, p->rs.off, p->rs.leafseg, Z64,
        zin_pitch, dc, Zhat, n_img, zrows, x, anchors, H, W, geo);
    FEPLL_LAUNCH();
    return kOk;
  };
  auto launch_split = [&](auto nt) -> int {
    constexpr int N = decltype(nt)::value;
    if constexpr (N % 2 == 0 && N <= 8) return launch(wn::wiener_dmma_kernel<N, 64, 2, 16, false, ZT, true>);
    return kDataError;
  };
#define FEPLL_WN_CASE(N)                                                   \
  case N:                                                                  \
    if (split) return launch_split(std::integral_constant<int, N>{});      \
    return big ? launch(wn::wiener_dmma_kernel<N, 128, 2, 16, false, ZT>)      \
               : ns == 4 ? launch(wn::wiener_dmma_kernel<N, 64, 4, 16, false, ZT>) \
               : rw == 8 ? launch(wn::wiener_dmma_kernel<N, 64, 2, 8, false, ZT>)  \
                         : launch(wn::wiener_dmma_kernel<N, 64, 2, 16, false, ZT>);
  if constexpr (sizeof(ZT) == 8) {
    if (xw) return launch(wn::wiener_dmma_kernel<8, 64, 2, 8, true>);
  }
  switch (nt2) {
    FEPLL_WN_CASE(1)
    FEPLL_WN_CASE(2)
    FEPLL_WN_CASE(4)
    FEPLL_WN_CASE(5)
    FEPLL_WN_CASE(7)
    FEPLL_WN_CASE(8)
    FEPLL_WN_CASE(11)
    FEPLL_WN_CASE(13)
    FEPLL_WN_CASE(16)
    default: break;
  }
#undef FEPLL_WN_CASE
  set_error("wiener: unsupported patch size for the DMMA kernel");
  return kDataError;
}

int wiener_dmma(Plan* p, int t, const double* Z64, const double* dc, double* Zhat, int n_img,
                int zrows, const double* x, const int32_t* anchors, int H, int W, cudaStream_t st) {
  return wiener_dmma_t<double>(p, t, Z64, p->v.P, dc, Zhat, n_img, zrows, x, anchors, H, W, st);
}

// FP32-state mode: FP32 patch rows in (pitch z32_pitch), FP32 est + dc out
int wiener_dmma_f32(Plan* p, int t, const float* Z32, int z32_pitch, const double* dc, float* Zhat,
                    int n_img, int zrows, const double* x, const int32_t* anchors, int H, int W,
                    cudaStream_t st) {
  return wiener_dmma_t<float>(p, t, Z32, z32_pitch, dc, Zhat, n_img, zrows, x, anchors, H, W, st);
}

bool wiener_dmma_supported(const Plan* p) {
  const int P = p->v.P;
  const int nt2 = (P + 7) / 8;
  const bool nt_ok = nt2 == 1 || nt2 == 2 || nt2 == 4 || nt2 == 5 || nt2 == 7 || nt2 == 8 ||
                     nt2 == 11 || nt2 == 13 || nt2 == 16;
  return P % 4 == 0 && P <= wn::kMaxP && p->max_model_rank <= wn::kMaxR && nt_ok;
}

}  // namespace fepll

extern "C" int fepll_debug_wiener_trace(void* device_buffer) {
  uint64_t* p = static_cast<uint64_t*>(device_buffer);
  return cudaMemcpyToSymbol(fepll::wn::g_trace, &p, sizeof(p)) == cudaSuccess ? 0 : 5;
}


