// Kernel (a): patch extraction with DC removal.
//
// Restates pkg/src/fepll/patches.py:167-183: window read row-major at each
// anchor, dc = _row_mean (pairwise fold, patches.py:153-164), stored = win - dc,
// all in FP64 so the patches are bit-identical to the reference's.  One warp
// per patch; the fold runs in a per-warp shared-memory row so its addition
// order is exactly the reference's for any P (odd widths fold their trailing
// column into the last slot).
#include "common.cuh"

namespace fepll {

constexpr int kExtractWarps = 8;

__global__ void __launch_bounds__(kExtractWarps * 32)
extract_kernel(const double* __restrict__ x, int batch, int H, int W, int side,
               const int32_t* __restrict__ anchors, int n, double* __restrict__ Z64,
               float* __restrict__ Z32, int z32_pitch, double* __restrict__ dc_out,
               double* __restrict__ sq_out) {
  __shared__ double buf[kExtractWarps][kMaxP];
  const int lane = lane_id();
  double* acc = buf[warp_id()];
  const int P = side * side;
  const int64_t total = (int64_t)batch * n;
  for (int64_t g = (int64_t)blockIdx.x * kExtractWarps + warp_id(); g < total;
       g += (int64_t)gridDim.x * kExtractWarps) {
    const int b = (int)(g / n);
    const int i = (int)(g - (int64_t)b * n);
    const int r0 = anchors[2 * i], c0 = anchors[2 * i + 1];
    const double* img = x + (int64_t)b * H * W;
    double win[kMaxP / 32];
#pragma unroll
    for (int k = 0; k < kMaxP / 32; ++k) {
      const int p = lane + 32 * k;
      if (p < P) {
        const int dr = p / side, dcol = p - dr * side;
        win[k] = img[(int64_t)(r0 + dr) * W + (c0 + dcol)];
        acc[p] = win[k];
      }
    }
    __syncwarp();
    // pairwise fold: acc[:h] + acc[h:2h], odd trailing column added to slot h-1
    for (int w = P; w > 1;) {
      const int h = w >> 1;
      double v[kMaxP / 64 + 1];
#pragma unroll
      for (int k = 0; k < kMaxP / 64 + 1; ++k) {
        const int p = lane + 32 * k;
        if (p < h) v[k] = acc[p] + acc[p + h];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kMaxP / 64 + 1; ++k) {
        const int p = lane + 32 * k;
        if (p < h) acc[p] = v[k];
      }
      __syncwarp();
      if ((w & 1) && lane == 0) acc[h - 1] += acc[w - 1];
      __syncwarp();
      w = h;
    }
    const double dc = acc[0] / (double)P;
    __syncwarp();
    double sq = 0.0;
    double* zrow = Z64 ? Z64 + g * P : nullptr;
    float* frow = Z32 ? Z32 + g * z32_pitch : nullptr;
#pragma unroll
    for (int k = 0; k < kMaxP / 32; ++k) {
      const int p = lane + 32 * k;
      if (p < P) {
        const double z = win[k] - dc;
        sq = fma(z, z, sq);
        if (zrow) zrow[p] = z;
        if (frow) frow[p] = (float)z;
      }
    }
    if (frow)
      for (int p = P + lane; p < z32_pitch; p += 32) frow[p] = 0.0f;
    sq = warp_sum(sq);
    if (lane == 0) {
      if (dc_out) dc_out[g] = dc;
      if (sq_out) sq_out[g] = sq;
    }
  }
}

// Fast path for power-of-two sides (P = 16, 64, 256): a group of `side`
// lanes owns one patch, lane r holds window row r in registers.  For
// P = side^2 with side = 2^k the reference's halvings of the flattened row
// (patches.py:156-163) first add row r + side/2, side/4, ... (k shuffle
// steps down the lane group) and then fold the surviving row in registers —
// the identical sequence of FP64 additions, so dc stays bitwise equal.
template <int SIDE>
__global__ void __launch_bounds__(256)
extract_pow2_kernel(const double* __restrict__ x, int batch, int H, int W,
                    const int32_t* __restrict__ anchors, int n, double* __restrict__ Z64,
                    float* __restrict__ Z32, int z32_pitch, double* __restrict__ dc_out,
                    double* __restrict__ sq_out) {
  constexpr int P = SIDE * SIDE;
  constexpr int PER_WARP = 32 / SIDE;  // patches per warp (SIDE <= 32)
  const int lane = threadIdx.x & 31;
  const int r = lane % SIDE;           // window row owned by this lane
  const int64_t total = (int64_t)batch * n;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * PER_WARP < total;
       w += warps) {
    const int64_t g = w * PER_WARP + lane / SIDE;
    const bool valid = g < total;
    double v[SIDE];
    if (valid) {
      const int b = (int)(g / n);
      const int i = (int)(g - (int64_t)b * n);
      const int pr = anchors[2 * i], pc = anchors[2 * i + 1];
      const double* src = x + ((int64_t)b * H + pr + r) * W + pc;
#pragma unroll
      for (int c = 0; c < SIDE; ++c) v[c] = __ldg(src + c);
    } else {
#pragma unroll
      for (int c = 0; c < SIDE; ++c) v[c] = 0.0;
    }
    // row halvings: lane r adds lane r + h for h = SIDE/2, ..., 1
    double acc[SIDE];
#pragma unroll
    for (int c = 0; c < SIDE; ++c) acc[c] = v[c];
#pragma unroll
    for (int h = SIDE / 2; h >= 1; h >>= 1) {
#pragma unroll
      for (int c = 0; c < SIDE; ++c) {
        const double o = __shfl_down_sync(0xffffffffu, acc[c], h, SIDE);
        if (r < h) acc[c] = acc[c] + o;
      }
    }
    // column halvings inside row 0
#pragma unroll
    for (int h = SIDE / 2; h >= 1; h >>= 1)
#pragma unroll
      for (int c = 0; c < h; ++c) acc[c] = acc[c] + acc[c + h];
    const double dc = __shfl_sync(0xffffffffu, acc[0], 0, SIDE) / (double)P;
    double sq = 0.0;
    if (valid) {
      double* zrow = Z64 ? Z64 + g * P + r * SIDE : nullptr;
      float* frow = Z32 ? Z32 + g * z32_pitch + r * SIDE : nullptr;
#pragma unroll
      for (int c = 0; c < SIDE; ++c) {
        const double z = v[c] - dc;
        sq = fma(z, z, sq);
        if (zrow) zrow[c] = z;
        if (frow) frow[c] = (float)z;
      }
      if (frow && r == 0)
        for (int p = P; p < z32_pitch; ++p) Z32[g * z32_pitch + p] = 0.0f;
    }
#pragma unroll
    for (int h = SIDE / 2; h >= 1; h >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, h, SIDE);
    if (valid && r == 0) {
      if (dc_out) dc_out[g] = dc;
      if (sq_out) sq_out[g] = sq;
    }
  }
}

}  // namespace fepll

extern "C" int fepll_extract(const double* x, int32_t batch, int32_t H, int32_t W, int32_t side,
                             const int32_t* anchors, int32_t n, double* Z64, float* Z32,
                             int32_t z32_pitch, double* dc, double* sq, void* stream) {
  using namespace fepll;
  FEPLL_REQUIRE(x && anchors && batch >= 1 && n >= 0, "extract: bad arguments");
  FEPLL_REQUIRE(side >= 1 && side * side <= kMaxP, "extract: patch side out of range");
  FEPLL_REQUIRE(H >= side && W >= side, "extract: image smaller than the patch");
  FEPLL_REQUIRE(Z32 == nullptr || z32_pitch >= side * side, "extract: Z32 pitch below P");
  if (n == 0) return kOk;
  const int64_t total = (int64_t)batch * n;
  cudaStream_t st = (cudaStream_t)stream;
  if (side == 8 || side == 4 || side == 16) {
    const int per_warp = 32 / side;
    const int64_t warps = (total + per_warp - 1) / per_warp;
    const int grid = grid_for(warps, 8, 148 * 32);
    if (side == 8)
      extract_pow2_kernel<8><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
    else if (side == 4)
      extract_pow2_kernel<4><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
    else
      extract_pow2_kernel<16><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
  } else {
    extract_kernel<<<grid_for(total, kExtractWarps, 148 * 64), kExtractWarps * 32, 0, st>>>(
        x, batch, H, W, side, anchors, n, Z64, Z32, z32_pitch, dc, sq);
  }
  FEPLL_LAUNCH();
  return kOk;
}
