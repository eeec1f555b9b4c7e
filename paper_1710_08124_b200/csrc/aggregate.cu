// Kernel (d) + fused pixel-diagonal kernel (e).
//
// Aggregation restates pkg/src/fepll/patches.py:198-222: x~(p) = sum over
// covering patches of (zhat + dc) / count (dc == NULL: the Wiener kernels
// already wrote zhat + dc, rounded exactly as here), with the lo == hi rule returning
// the common value verbatim.  np.bincount accumulates each pixel's values in
// increasing patch index; this kernel gathers, per pixel, the candidate
// anchors of the nominal grid in the same (row-major) order, so the FP64
// sums are bit-identical — no atomics, run-to-run deterministic.
//
// Strip mode (one image split across ranks by pixel rows, DESIGN.md
// "Multi-GPU"): the local image is global rows [row0, row0 + H) of an image
// of H_glob rows, the local patch arrays hold the anchors of global nominal
// rows a_first.., and only local rows [r_begin, r_end) are produced.  The
// candidate set and its order are the global ones, so every produced pixel
// is bit-identical to the unsplit run.
//
// For pixel-diagonal operators the image update of
// pkg/src/fepll/operators.py:281-287 (x = (A^T y + bs2 x~) / (diag + bs2)) is
// applied in the same pass with explicit round-to-nearest multiply/add (no
// FMA contraction) so it is bit-identical to numpy's two-step evaluation.
#include <climits>

#include "common.cuh"

namespace fepll {

__device__ __forceinline__ int ceil_div_floor0(int num, int s) {
  return num <= 0 ? 0 : (num + s - 1) / s;
}

struct GridGeo {
  const int32_t* anchors;
  int n_rows, n_cols, s, half, side, W;
  int row0, H_glob, a_first;
};

// Visit the anchors covering global pixel (r, c) in ascending patch index —
// np.bincount's accumulation order (patches.py:213-220): candidate nominal
// rows a with a*s in [r-side+1-half, r+half] (a <= n_rows-2), then the
// clamped last row; within a row the candidate columns likewise, then the
// last column.  fn(local patch index, dr, dcol).
template <class F>
__device__ __forceinline__ void for_each_cover(const GridGeo& g, int r, int c, F&& fn) {
  const int side = g.side, s = g.s, half = g.half;
  const int last_r = g.H_glob - side, last_c = g.W - side;
  const int a_lo = ceil_div_floor0(r - side + 1 - half, s);
  const int a_hi = min(g.n_rows - 2, (r + half) / s);
  const int b_lo = ceil_div_floor0(c - side + 1 - half, s);
  const int b_hi = min(g.n_cols - 2, (c + half) / s);
  const bool last_row_ok = last_r <= r + half;  // always >= r-side+1-half
  const bool last_col_ok = last_c <= c + half;
  auto visit = [&](int ia, int ib) {
    const int i = (ia - g.a_first) * g.n_cols + ib;  // local patch index
    const int dr = r - (g.row0 + g.anchors[2 * i]), dcol = c - g.anchors[2 * i + 1];
    if ((unsigned)dr < (unsigned)side && (unsigned)dcol < (unsigned)side) fn(i, dr, dcol);
  };
  auto visit_row = [&](int ia) {
    for (int ib = b_lo; ib <= b_hi; ++ib) visit(ia, ib);
    if (last_col_ok) visit(ia, g.n_cols - 1);
  };
  for (int ia = a_lo; ia <= a_hi; ++ia) visit_row(ia);
  if (last_row_ok) visit_row(g.n_rows - 1);
}

// x~ (with the lo == hi rule) and the fused pixel update for one pixel
__device__ __forceinline__ void finish_pixel(double sum, double lo, double hi, int count,
                                             int64_t pix, const double* aty, const double* diag,
                                             double bs2, int kind, double* x_out, double* xt_out,
                                             int32_t* status) {
  double xt;
  if (count == 0) {
    atomicOr(status, 1);
    xt = 0.0;
  } else {
    xt = (lo == hi) ? lo : __ddiv_rn(sum, (double)count);
  }
  if (xt_out) xt_out[pix] = xt;
  const double at = aty ? aty[pix] : 0.0;
  const double rhs = __dadd_rn(at, __dmul_rn(bs2, xt));
  if (kind == 0) {
    const double dg = diag ? diag[pix] : 1.0;
    const double x = __ddiv_rn(rhs, __dadd_rn(dg, bs2));
    if (!isfinite(x)) atomicOr(status, 2);
    if (x_out) x_out[pix] = x;
  } else if (x_out) {
    x_out[pix] = rhs;
  }
}

template <typename ZT>
__global__ void __launch_bounds__(256)
aggregate_kernel(const ZT* __restrict__ Zhat, const double* __restrict__ dc, GridGeo geo,
                 int batch, int H, const double* __restrict__ aty,
                 const double* __restrict__ diag, double bs2, int kind,
                 double* __restrict__ x_out, double* __restrict__ xt_out, int32_t* status,
                 int n_local_rows, int r_begin) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r_loc = r_begin + blockIdx.y;
  const int b = blockIdx.z;
  const int W = geo.W;
  if (c >= W) return;
  const int P = geo.side * geo.side;
  const int64_t gbase = (int64_t)b * n_local_rows * geo.n_cols;
  double sum = 0.0, lo = INFINITY, hi = -INFINITY;
  int count = 0;
  for_each_cover(geo, geo.row0 + r_loc, c, [&](int i, int dr, int dcol) {
    const int64_t g = gbase + i;
    const double z = (double)Zhat[g * P + dr * geo.side + dcol];
    const double v = dc ? __dadd_rn(z, dc[g]) : z;  // dc == NULL: Zhat holds est + dc
    sum += v;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
    ++count;
  });
  finish_pixel(sum, lo, hi, count, ((int64_t)b * H + r_loc) * W + c, aty, diag, bs2, kind, x_out,
               xt_out, status);
}

// ---- cover lists: the grid is shared by every image of a batch, so the
// covering (patch, offset) entries of each pixel are enumerated once per
// sampling plan, as CSR in ascending patch order: entry = i << 8 | offset.
__global__ void cover_count_kernel(GridGeo geo, int r_begin, int rows, int32_t* __restrict__ counts) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)rows * geo.W) return;
  const int r_loc = r_begin + (int)(p / geo.W), c = (int)(p % geo.W);
  int k = 0;
  for_each_cover(geo, geo.row0 + r_loc, c, [&](int, int, int) { ++k; });
  counts[p] = k;
}

__global__ void cover_fill_kernel(GridGeo geo, int r_begin, int rows, const int32_t* __restrict__ ptr,
                                  int32_t* __restrict__ entries) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)rows * geo.W) return;
  const int r_loc = r_begin + (int)(p / geo.W), c = (int)(p % geo.W);
  int32_t* out = entries + ptr[p];
  for_each_cover(geo, geo.row0 + r_loc, c, [&](int i, int dr, int dcol) {
    *out++ = (i << 8) | (dr * geo.side + dcol);
  });
}

// exclusive scan of counts[0..n) into ptr[0..n] (ptr[n] = total): block
// sums, one-block scan of the sums, block-local scans
__global__ void scan_blocks_kernel(const int32_t* __restrict__ counts, int64_t n, int32_t* __restrict__ bsum) {
  __shared__ int32_t red[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  int v = i < n ? counts[i] : 0;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    int w = red[threadIdx.x];
    w = warp_sum(w);
    if (threadIdx.x == 0) bsum[blockIdx.x] = w;
  }
}

__global__ void scan_sums_kernel(int32_t* bsum, int nb) {
  // single block of 1024 threads, sequential chunks
  __shared__ int32_t carry;
  __shared__ int32_t tmp[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    tmp[threadIdx.x] = i < nb ? bsum[i] : 0;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int v = threadIdx.x >= off ? tmp[threadIdx.x - off] : 0;
      __syncthreads();
      tmp[threadIdx.x] += v;
      __syncthreads();
    }
    if (i < nb) bsum[i] = carry + tmp[threadIdx.x] - (i < nb ? bsum[i] : 0);
    __syncthreads();
    if (threadIdx.x == 1023) carry += tmp[1023];
    __syncthreads();
  }
}

__global__ void scan_apply_kernel(const int32_t* __restrict__ counts, int64_t n,
                                  const int32_t* __restrict__ bsum, int32_t* __restrict__ ptr) {
  __shared__ int32_t tmp[1024];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int v = i < n ? counts[i] : 0;
  tmp[threadIdx.x] = v;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int u = threadIdx.x >= off ? tmp[threadIdx.x - off] : 0;
    __syncthreads();
    tmp[threadIdx.x] += u;
    __syncthreads();
  }
  if (i < n) ptr[i] = bsum[blockIdx.x] + tmp[threadIdx.x] - v;
  if (i == n - 1) ptr[n] = bsum[blockIdx.x] + tmp[threadIdx.x];
}

// Gather over the cover list.  A thread owns one pixel for a group of the
// batch's images (blockIdx.z): the pixel's cover entries (the plan is the
// batch's) are decoded once into element offsets held in registers, then
// each image costs its Zhat loads, the ordered sum and the pixel update —
// the gather is issue-bound, so the per-image instruction count is what is
// minimised, and occupancy (latency hiding) matters more than loads in
// flight per thread: measured on B200, 64 registers / 4 blocks per SM and
// one image at a time beat several images per pass (those run slower).
// Per image the result is aggregate_kernel's:
//  * the sum runs over the entries in ascending patch order from 0.0;
//  * lo == hi (patches.py:221) is "every value equals the first" (NaN
//    compares unequal, so a NaN still reaches the sum);
//  * sum / count for a power-of-two count is the exact product with 1/count.
constexpr int kCoverThreads = 256;
constexpr int kCoverRegEntries = 9;   // entries decoded into registers (more: generic loop)
constexpr int kCoverImgPerBlock = 64; // images per block (blockIdx.z groups; per-block setup is
                                      // three dependent loads, amortised over the images)

__device__ __forceinline__ void pixel_update(double xt, int64_t pix, const double* aty,
                                             const double* diag, double bs2, int kind,
                                             double* x_out, double* xt_out, int32_t* status) {
  if (xt_out) xt_out[pix] = xt;
  const double at = aty ? aty[pix] : 0.0;
  const double rhs = __dadd_rn(at, __dmul_rn(bs2, xt));
  if (kind == 0) {
    const double dg = diag ? diag[pix] : 1.0;
    const double x = __ddiv_rn(rhs, __dadd_rn(dg, bs2));
    if (!isfinite(x)) atomicOr(status, 2);
    if (x_out) x_out[pix] = x;
  } else if (x_out) {
    x_out[pix] = rhs;
  }
}

template <bool kDc, int NB, bool CG, typename ZT>
__global__ void __launch_bounds__(kCoverThreads, 4)  // 64 registers: 4 blocks per SM
aggregate_cover_kernel(const ZT* __restrict__ Zhat, const double* __restrict__ dc,
                       const int32_t* __restrict__ ptr, const int32_t* __restrict__ entries, int P,
                       int n_local, int zrows, int batch, int H, int W, int r_begin,
                       const double* __restrict__ aty, const double* __restrict__ diag, double bs2,
                       int kind, double* __restrict__ x_out, double* __restrict__ xt_out,
                       int32_t* status, int ipb) {
  const int c = blockIdx.x * kCoverThreads + threadIdx.x;
  if (c >= W) return;
  const int64_t p = (int64_t)blockIdx.y * W + c;  // pixel within the cover rows
  const int e0 = __ldg(ptr + p), cnt = __ldg(ptr + p + 1) - e0;
  const int64_t pix0 = (int64_t)(r_begin + blockIdx.y) * W + c;
  const int64_t img = (int64_t)H * W;
  const int64_t zimg = (int64_t)zrows * P;  // Zhat elements per image (padded pitch)
  const int b_begin = blockIdx.z * ipb;
  const int b_end = min(batch, b_begin + ipb);
  if (cnt == 0) {
    atomicOr(status, 1);
    for (int b = b_begin; b < b_end; ++b)
      pixel_update(0.0, b * img + pix0, aty, diag, bs2, kind, x_out, xt_out, status);
    return;
  }
  const bool pow2 = (cnt & (cnt - 1)) == 0;
  const double inv = 1.0 / (double)cnt;  // exact when pow2
  if (cnt <= kCoverRegEntries) {
    int off[kCoverRegEntries];
    int dco[kCoverRegEntries];
#pragma unroll
    for (int q = 0; q < kCoverRegEntries; ++q) {
      const int v = q < cnt ? __ldg(entries + e0 + q) : 0;
      off[q] = (v >> 8) * P + (v & 255);
      dco[q] = v >> 8;
    }
    for (int b = b_begin; b < b_end; b += NB) {
      // NB images' loads in flight before the first sum; the Zhat sectors
      // are used once each, so they skip L1 (CG) unless g_cover_l1
      double v[NB][kCoverRegEntries];
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const ZT* zb = Zhat + (b + k) * zimg;
#pragma unroll
        for (int q = 0; q < kCoverRegEntries; ++q)
          if (q < cnt && (k == 0 || b + k < b_end)) {
            v[k][q] = CG ? (double)__ldcg(zb + off[q]) : (double)__ldg(zb + off[q]);
            if (kDc) v[k][q] = __dadd_rn(v[k][q], __ldg(dc + (int64_t)(b + k) * n_local + dco[q]));
          }
      }
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        if (k > 0 && b + k >= b_end) break;
        double sum = 0.0 + v[k][0];
        bool same = true;
#pragma unroll
        for (int q = 1; q < kCoverRegEntries; ++q)
          if (q < cnt) {
            sum += v[k][q];
            same = same && v[k][q] == v[k][0];
          }
        const double xt = same ? v[k][0] : pow2 ? sum * inv : __ddiv_rn(sum, (double)cnt);
        pixel_update(xt, (b + k) * img + pix0, aty, diag, bs2, kind, x_out, xt_out, status);
      }
    }
  } else {
    for (int b = b_begin; b < b_end; ++b) {
      const ZT* zb = Zhat + b * zimg;
      double sum = 0.0, v0 = 0.0;
      bool same = true;
      for (int q = 0; q < cnt; ++q) {
        const int e = __ldg(entries + e0 + q);
        double v = (double)__ldg(zb + (int64_t)(e >> 8) * P + (e & 255));
        if (kDc) v = __dadd_rn(v, __ldg(dc + (int64_t)b * n_local + (e >> 8)));
        if (q == 0) v0 = v;
        sum += v;
        same = same && v == v0;
      }
      const double xt = same ? v0 : pow2 ? sum * inv : __ddiv_rn(sum, (double)cnt);
      pixel_update(xt, b * img + pix0, aty, diag, bs2, kind, x_out, xt_out, status);
    }
  }
}

// Single-image form (row strips, large single images): one pixel per thread
// and nothing to amortise the entry decode over, so the kernel is the
// ptr -> entries -> Zhat chain of dependent loads; kept to 32 registers for
// full occupancy (twice the chains in flight of the batched kernel).
template <bool kDc, typename ZT>
__global__ void __launch_bounds__(kCoverThreads, 8)
aggregate_cover1_kernel(const ZT* __restrict__ Zhat, const double* __restrict__ dc,
                        const int32_t* __restrict__ ptr, const int32_t* __restrict__ entries,
                        int P, int W, int r_begin, const double* __restrict__ aty,
                        const double* __restrict__ diag, double bs2, int kind,
                        double* __restrict__ x_out, double* __restrict__ xt_out, int32_t* status,
                        int64_t zimg = 0, int64_t img = 0, int n_local = 0) {
  const int c = blockIdx.x * kCoverThreads + threadIdx.x;
  if (c >= W) return;
  // batches (blockIdx.z = image): one thread per (pixel, image) — every
  // image re-reads the plan's ptr / entries (L2-resident) for 2x the
  // resident threads of the per-pixel multi-image kernel
  Zhat += (int64_t)blockIdx.z * zimg;
  if (kDc) dc += (int64_t)blockIdx.z * n_local;
  const int64_t p = (int64_t)blockIdx.y * W + c;
  const int e0 = __ldg(ptr + p), cnt = __ldg(ptr + p + 1) - e0;
  const int64_t pix = (int64_t)blockIdx.z * img + (int64_t)(r_begin + blockIdx.y) * W + c;
  if (cnt == 0) {
    atomicOr(status, 1);
    pixel_update(0.0, pix, aty, diag, bs2, kind, x_out, xt_out, status);
    return;
  }
  double sum = 0.0, v0 = 0.0;
  bool same = true;
  if (cnt <= 4) {
    int e[4];
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) e[q] = q < cnt ? __ldg(entries + e0 + q) : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < cnt) {
        v[q] = (double)__ldg(Zhat + (int64_t)(e[q] >> 8) * P + (e[q] & 255));
        if (kDc) v[q] = __dadd_rn(v[q], __ldg(dc + (e[q] >> 8)));
      }
    v0 = v[0];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < cnt) {
        sum += v[q];
        same = same && v[q] == v0;
      }
  } else {
    for (int q = 0; q < cnt; ++q) {
      const int e = __ldg(entries + e0 + q);
      double v = (double)__ldg(Zhat + (int64_t)(e >> 8) * P + (e & 255));
      if (kDc) v = __dadd_rn(v, __ldg(dc + (e >> 8)));
      if (q == 0) v0 = v;
      sum += v;
      same = same && v == v0;
    }
  }
  const bool pow2 = (cnt & (cnt - 1)) == 0;
  const double xt = same ? v0 : pow2 ? sum * (1.0 / (double)cnt) : __ddiv_rn(sum, (double)cnt);
  pixel_update(xt, pix, aty, diag, bs2, kind, x_out, xt_out, status);
}

}  // namespace fepll

namespace fepll {
template <typename ZT>
static int aggregate_strip_impl(const ZT* Zhat, const double* dc, const int32_t* anchors,
                                     int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                                     int32_t side, int32_t batch, int32_t H, int32_t W,
                                     int32_t row0, int32_t H_glob, int32_t a_first,
                                     int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                                     const double* aty, const double* diag, double bs2, int32_t kind,
                                     double* x_out, double* xtilde_out, int32_t* status, void* stream) {
  FEPLL_REQUIRE(Zhat && anchors && status, "aggregate: bad arguments");
  FEPLL_REQUIRE(n_rows >= 1 && n_cols >= 1 && spacing >= 1 && side >= 1 && half >= 0,
                "aggregate: bad grid geometry");
  FEPLL_REQUIRE(H >= 1 && W >= side && batch >= 1 && H_glob >= side, "aggregate: bad image dims");
  FEPLL_REQUIRE(row0 >= 0 && row0 + H <= H_glob, "aggregate: strip outside the image");
  FEPLL_REQUIRE(0 <= r_begin && r_begin <= r_end && r_end <= H, "aggregate: output rows outside the strip");
  FEPLL_REQUIRE(a_first >= 0 && n_local_rows >= 1 && a_first + n_local_rows <= n_rows,
                "aggregate: local anchor rows outside the grid");
  FEPLL_REQUIRE(kind == 0 || kind == 1, "aggregate: unknown kind");
  FEPLL_REQUIRE(H <= 65535 && batch <= 65535, "aggregate: image too tall for the launch grid");
  if (r_end == r_begin) return kOk;
  dim3 grid((W + 255) / 256, r_end - r_begin, batch);
  const GridGeo geo{anchors, n_rows, n_cols, spacing, half, side, W, row0, H_glob, a_first};
  aggregate_kernel<ZT><<<grid, 256, 0, (cudaStream_t)stream>>>(
      Zhat, dc, geo, batch, H, aty, diag, bs2, kind, x_out, xtilde_out, status, n_local_rows,
      r_begin);
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll

extern "C" int fepll_aggregate_strip(const double* Zhat, const double* dc, const int32_t* anchors,
                                     int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                                     int32_t side, int32_t batch, int32_t H, int32_t W,
                                     int32_t row0, int32_t H_glob, int32_t a_first,
                                     int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                                     const double* aty, const double* diag, double bs2, int32_t kind,
                                     double* x_out, double* xtilde_out, int32_t* status, void* stream) {
  return fepll::aggregate_strip_impl(Zhat, dc, anchors, n_rows, n_cols, spacing, half, side, batch, H, W,
                                     row0, H_glob, a_first, n_local_rows, r_begin, r_end, aty, diag, bs2,
                                     kind, x_out, xtilde_out, status, stream);
}

extern "C" int fepll_aggregate_strip_f32(const float* Zhat, const double* dc, const int32_t* anchors,
                                         int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                                         int32_t side, int32_t batch, int32_t H, int32_t W,
                                         int32_t row0, int32_t H_glob, int32_t a_first,
                                         int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                                         const double* aty, const double* diag, double bs2, int32_t kind,
                                         double* x_out, double* xtilde_out, int32_t* status, void* stream) {
  return fepll::aggregate_strip_impl(Zhat, dc, anchors, n_rows, n_cols, spacing, half, side, batch, H, W,
                                     row0, H_glob, a_first, n_local_rows, r_begin, r_end, aty, diag, bs2,
                                     kind, x_out, xtilde_out, status, stream);
}

extern "C" int fepll_aggregate(const double* Zhat, const double* dc, const int32_t* anchors,
                               int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                               int32_t side, int32_t batch, int32_t H, int32_t W,
                               const double* aty, const double* diag, double bs2, int32_t kind,
                               double* x_out, double* xtilde_out, int32_t* status, void* stream) {
  return fepll_aggregate_strip(Zhat, dc, anchors, n_rows, n_cols, spacing, half, side, batch, H, W,
                               0, H, 0, n_rows, 0, H, aty, diag, bs2, kind, x_out, xtilde_out,
                               status, stream);
}

extern "C" int64_t fepll_cover_scratch_ints(int64_t n_pixels) {
  return n_pixels + (n_pixels + 1023) / 1024 + 1;
}

extern "C" int fepll_cover_build(const int32_t* anchors, int32_t n_rows, int32_t n_cols,
                                 int32_t spacing, int32_t half, int32_t side, int32_t W,
                                 int32_t row0, int32_t H_glob, int32_t a_first,
                                 int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                                 int32_t* ptr, int32_t* entries, int64_t entries_cap,
                                 int32_t* scratch, void* stream) {
  using namespace fepll;
  FEPLL_REQUIRE(anchors && ptr && entries && scratch, "cover_build: bad arguments");
  FEPLL_REQUIRE(side * side <= 256 && side >= 1 && spacing >= 1 && half >= 0,
                "cover_build: bad grid geometry");
  FEPLL_REQUIRE((int64_t)n_local_rows * n_cols < (int64_t(1) << 23),
                "cover_build: more than 2^23 patches per image");
  FEPLL_REQUIRE(0 <= r_begin && r_begin <= r_end && row0 >= 0 && row0 + r_end <= H_glob,
                "cover_build: rows outside the image");
  const int rows = r_end - r_begin;
  const int64_t npx = (int64_t)rows * W;
  if (npx == 0) return kOk;
  cudaStream_t st = (cudaStream_t)stream;
  const GridGeo geo{anchors, n_rows, n_cols, spacing, half, side, W, row0, H_glob, a_first};
  int32_t* counts = scratch;
  int32_t* bsum = scratch + npx;
  const int64_t nb = (npx + 1023) / 1024;
  FEPLL_REQUIRE(nb < (int64_t(1) << 31), "cover_build: image too large");
  cover_count_kernel<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(geo, r_begin, rows, counts);
  FEPLL_LAUNCH();
  scan_blocks_kernel<<<(unsigned)nb, 1024, 0, st>>>(counts, npx, bsum);
  FEPLL_LAUNCH();
  scan_sums_kernel<<<1, 1024, 0, st>>>(bsum, (int)nb);
  FEPLL_LAUNCH();
  scan_apply_kernel<<<(unsigned)nb, 1024, 0, st>>>(counts, npx, bsum, ptr);
  FEPLL_LAUNCH();
  // every patch covers exactly P pixels of the full image; a strip holds
  // at most its patches' P each
  FEPLL_REQUIRE(entries_cap >= (int64_t)n_local_rows * n_cols * side * side,
                "cover_build: entry buffer below n_local * P");
  cover_fill_kernel<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(geo, r_begin, rows, ptr, entries);
  FEPLL_LAUNCH();
  return kOk;
}

namespace fepll {
template <typename ZT>
static int aggregate_cover_impl(const ZT* Zhat, const double* dc, const int32_t* ptr,
                                     const int32_t* entries, int32_t P, int32_t n_local,
                                     int32_t zhat_rows,
                                     int32_t batch, int32_t H, int32_t W, int32_t r_begin,
                                     int32_t r_end, const double* aty, const double* diag,
                                     double bs2, int32_t kind, double* x_out, double* xtilde_out,
                                     int32_t* status, void* stream, int variant = 0) {
  FEPLL_REQUIRE(Zhat && ptr && entries && status, "aggregate_cover: bad arguments");
  FEPLL_REQUIRE(kind == 0 || kind == 1, "aggregate_cover: unknown kind");
  FEPLL_REQUIRE(zhat_rows >= n_local, "aggregate_cover: Zhat rows per image below n_local");
  FEPLL_REQUIRE(0 <= r_begin && r_begin <= r_end && r_end <= H && batch >= 1,
                "aggregate_cover: bad rows");
  if (r_end == r_begin) return kOk;
  FEPLL_REQUIRE(r_end - r_begin <= 65535, "aggregate_cover: strip taller than the launch grid");
  const int ipb = kCoverImgPerBlock;
  FEPLL_REQUIRE((int64_t)n_local * P < (int64_t(1) << 31), "aggregate_cover: image patch array above 2^31 elements");
  dim3 grid((unsigned)((W + kCoverThreads - 1) / kCoverThreads), r_end - r_begin,
            (unsigned)((batch + ipb - 1) / ipb));
  if (batch == 1 || variant == 1) {
    FEPLL_REQUIRE(batch <= 65535, "aggregate_cover: batch above the launch grid");
    dim3 g1((unsigned)((W + kCoverThreads - 1) / kCoverThreads), r_end - r_begin, batch);
    auto k1 = dc ? aggregate_cover1_kernel<true, ZT> : aggregate_cover1_kernel<false, ZT>;
    k1<<<g1, kCoverThreads, 0, (cudaStream_t)stream>>>(Zhat, dc, ptr, entries, P, W, r_begin, aty,
                                                       diag, bs2, kind, x_out, xtilde_out, status,
                                                       (int64_t)zhat_rows * P, (int64_t)H * W, n_local);
    FEPLL_LAUNCH();
    return kOk;
  }
  // one image per pass, Zhat loads past L1 (measured: two images per pass
  // spill at 64 registers and run 15 % slower; L1-cached loads 2-3 % slower)
  auto kernel = dc ? aggregate_cover_kernel<true, 1, true, ZT> : aggregate_cover_kernel<false, 1, true, ZT>;
  kernel<<<grid, kCoverThreads, 0, (cudaStream_t)stream>>>(
      Zhat, dc, ptr, entries, P, n_local, zhat_rows, batch, H, W, r_begin, aty, diag, bs2, kind, x_out,
      xtilde_out, status, ipb);
  FEPLL_LAUNCH();
  return kOk;
}
}  // namespace fepll

extern "C" int fepll_aggregate_cover(const double* Zhat, const double* dc, const int32_t* ptr,
                                     const int32_t* entries, int32_t P, int32_t n_local,
                                     int32_t zhat_rows,
                                     int32_t batch, int32_t H, int32_t W, int32_t r_begin,
                                     int32_t r_end, const double* aty, const double* diag,
                                     double bs2, int32_t kind, double* x_out, double* xtilde_out,
                                     int32_t* status, void* stream) {
  return fepll::aggregate_cover_impl(Zhat, dc, ptr, entries, P, n_local, zhat_rows, batch, H, W, r_begin,
                                     r_end, aty, diag, bs2, kind, x_out, xtilde_out, status, stream);
}

extern "C" int fepll_aggregate_cover_f32(const float* Zhat, const double* dc, const int32_t* ptr,
                                         const int32_t* entries, int32_t P, int32_t n_local,
                                         int32_t zhat_rows,
                                         int32_t batch, int32_t H, int32_t W, int32_t r_begin,
                                         int32_t r_end, const double* aty, const double* diag,
                                         double bs2, int32_t kind, double* x_out, double* xtilde_out,
                                         int32_t* status, void* stream) {
  return fepll::aggregate_cover_impl(Zhat, dc, ptr, entries, P, n_local, zhat_rows, batch, H, W, r_begin,
                                     r_end, aty, diag, bs2, kind, x_out, xtilde_out, status, stream);
}

// fepll_aggregate_cover with an explicit batch kernel: variant 0 = one
// thread per pixel looping over the images (entries decoded once),
// 1 = one thread per (pixel, image).  Bitwise-identical results.
extern "C" int fepll_aggregate_cover_ex(const double* Zhat, const float* Zhat32, const double* dc,
                                        const int32_t* ptr, const int32_t* entries, int32_t P,
                                        int32_t n_local, int32_t zhat_rows, int32_t batch, int32_t H,
                                        int32_t W, int32_t r_begin, int32_t r_end, const double* aty,
                                        const double* diag, double bs2, int32_t kind, double* x_out,
                                        double* xtilde_out, int32_t* status, int32_t variant,
                                        void* stream) {
  FEPLL_REQUIRE((Zhat == nullptr) != (Zhat32 == nullptr), "aggregate_cover_ex: exactly one of Zhat / Zhat32");
  FEPLL_REQUIRE(variant == 0 || variant == 1, "aggregate_cover_ex: unknown variant");
  if (Zhat32)
    return fepll::aggregate_cover_impl(Zhat32, dc, ptr, entries, P, n_local, zhat_rows, batch, H, W, r_begin,
                                       r_end, aty, diag, bs2, kind, x_out, xtilde_out, status, stream, variant);
  return fepll::aggregate_cover_impl(Zhat, dc, ptr, entries, P, n_local, zhat_rows, batch, H, W, r_begin,
                                     r_end, aty, diag, bs2, kind, x_out, xtilde_out, status, stream, variant);
}
