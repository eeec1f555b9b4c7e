// Kernel (d) + fused pixel-diagonal kernel (e).
//
// Aggregation restates pkg/src/fepll/patches.py:198-222: x~(p) = sum over
// covering patches of (zhat + dc) / count, with the lo == hi rule returning
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
#include "common.cuh"

namespace fepll {

__device__ __forceinline__ int ceil_div_floor0(int num, int s) {
  return num <= 0 ? 0 : (num + s - 1) / s;
}

__global__ void __launch_bounds__(256)
aggregate_kernel(const double* __restrict__ Zhat, const double* __restrict__ dc,
                 const int32_t* __restrict__ anchors, int n_rows, int n_cols, int s, int half,
                 int side, int batch, int H, int W, const double* __restrict__ aty,
                 const double* __restrict__ diag, double bs2, int kind,
                 double* __restrict__ x_out, double* __restrict__ xt_out, int32_t* status,
                 int row0, int H_glob, int a_first, int n_local_rows, int r_begin) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r_loc = r_begin + blockIdx.y;
  const int r = row0 + r_loc;  // global row
  const int b = blockIdx.z;
  if (c >= W) return;
  const int P = side * side;
  const int n = n_local_rows * n_cols;  // local patches per image
  const int last_r = H_glob - side, last_c = W - side;
  // candidate nominal rows a with R_a in [r-side+1-half, r+half]
  const int a_lo = ceil_div_floor0(r - side + 1 - half, s);
  const int a_hi = min(n_rows - 2, (r + half) / s);
  const int b_lo = ceil_div_floor0(c - side + 1 - half, s);
  const int b_hi = min(n_cols - 2, (c + half) / s);
  const bool last_row_ok = last_r <= r + half;  // always >= r-side+1-half
  const bool last_col_ok = last_c <= c + half;
  const int64_t gbase = (int64_t)b * n;
  double sum = 0.0, lo = INFINITY, hi = -INFINITY;
  int count = 0;
  auto visit = [&](int ia, int ib) {
    const int i = (ia - a_first) * n_cols + ib;  // local patch index
    const int pr = row0 + anchors[2 * i], pc = anchors[2 * i + 1];
    const int dr = r - pr, dcol = c - pc;
    if ((unsigned)dr < (unsigned)side && (unsigned)dcol < (unsigned)side) {
      const int64_t g = gbase + i;
      const double v = __dadd_rn(Zhat[g * P + dr * side + dcol], dc[g]);
      sum += v;
      lo = fmin(lo, v);
      hi = fmax(hi, v);
      ++count;
    }
  };
  auto visit_row = [&](int ia) {
    for (int ib = b_lo; ib <= b_hi; ++ib) visit(ia, ib);
    if (last_col_ok) visit(ia, n_cols - 1);
  };
  // ascending patch index == np.bincount's accumulation order
  for (int ia = a_lo; ia <= a_hi; ++ia) visit_row(ia);
  if (last_row_ok) visit_row(n_rows - 1);
  const int64_t pix = ((int64_t)b * H + r_loc) * W + c;
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

}  // namespace fepll

extern "C" int fepll_aggregate_strip(const double* Zhat, const double* dc, const int32_t* anchors,
                                     int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                                     int32_t side, int32_t batch, int32_t H, int32_t W,
                                     int32_t row0, int32_t H_glob, int32_t a_first,
                                     int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                                     const double* aty, const double* diag, double bs2, int32_t kind,
                                     double* x_out, double* xtilde_out, int32_t* status, void* stream) {
  using namespace fepll;
  FEPLL_REQUIRE(Zhat && dc && anchors && status, "aggregate: bad arguments");
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
  aggregate_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      Zhat, dc, anchors, n_rows, n_cols, spacing, half, side, batch, H, W, aty, diag, bs2, kind,
      x_out, xtilde_out, status, row0, H_glob, a_first, n_local_rows, r_begin);
  FEPLL_LAUNCH();
  return kOk;
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
