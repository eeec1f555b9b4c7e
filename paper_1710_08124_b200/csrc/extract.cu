// Kernel (a): patch extraction with DC removal.
//
// Restates pkg/src/fepll/patches.py:167-183: window read row-major at each
// anchor, dc = _row_mean (pairwise fold, patches.py:153-164), stored = win - dc,
// all in FP64 so the patches are bit-identical to the reference's.  One warp
// per patch; the fold runs in a per-warp shared-memory row so its addition
// order is exactly the reference's for any P (odd widths fold their trailing
// column into the last slot).
#include <climits>

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

// Direct column variant for power-of-two sides: a group of SIDE lanes owns
// one patch, lane c holds window column c (SIDE rows) in registers, loaded
// straight from the image (the groups of a warp read overlapping spans of the
// same image rows, so the loads mostly hit L1).  The fold: row halvings in
// registers, then column halvings by shuffles (the same FP64 additions as patches.py:153-164).  Rows r, r + 1 of a column pair
// leave together after one lane-pair shuffle: the even lane stores row r's
// two columns, the odd lane row r + 1's, as one 16-byte (Z64) / 8-byte (Z32)
// store each — hence the alignment rule of paired_stores_ok().  No
// shared memory, no barriers: a few dozen instructions per patch (a staged
// shared-memory tile kernel measured several hundred, round 1).
template <int SIDE, int U, int MINB = 1>
__global__ void __launch_bounds__(256, MINB)
extract_cols_kernel(const double* __restrict__ x, int batch, int H, int W,
                    const int32_t* __restrict__ anchors, int n, double* __restrict__ Z64,
                    float* __restrict__ Z32, int z32_pitch, double* __restrict__ dc_out,
                    double* __restrict__ sq_out) {
  constexpr int P = SIDE * SIDE;
  constexpr int PER_WARP = 32 / SIDE;
  const int lane = threadIdx.x & 31;
  const int c = lane % SIDE;
  const int64_t total = (int64_t)batch * n;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  // U consecutive lane groups per warp iteration: all U x SIDE window loads
  // are issued before the first fold (the kernel is load-latency bound)
  for (int64_t w0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * U;
       w0 * PER_WARP < total; w0 += warps * U) {
    double v[U][SIDE];
    int64_t g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      g[u] = (w0 + u) * PER_WARP + lane / SIDE;
      if (g[u] < total) {
        const int b = (int)(g[u] / n);
        const int i = (int)(g[u] - (int64_t)b * n);
        const int2 a = __ldg(reinterpret_cast<const int2*>(anchors) + i);
        const double* src = x + ((int64_t)b * H + a.x) * W + a.y + c;
#pragma unroll
        for (int r = 0; r < SIDE; ++r) v[u][r] = __ldg(src + (int64_t)r * W);
      } else {
#pragma unroll
        for (int r = 0; r < SIDE; ++r) v[u][r] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool valid = g[u] < total;
      double acc[SIDE];
#pragma unroll
      for (int r = 0; r < SIDE; ++r) acc[r] = v[u][r];
#pragma unroll
      for (int h = SIDE / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int r = 0; r < h; ++r) acc[r] = acc[r] + acc[r + h];
      double col = acc[0];
#pragma unroll
      for (int h = SIDE / 2; h >= 1; h >>= 1) {
        const double o = __shfl_down_sync(0xffffffffu, col, h, SIDE);
        if (c < h) col = col + o;
      }
      const double dc = __shfl_sync(0xffffffffu, col, 0, SIDE) / (double)P;
      double sq = 0.0;
      double zz[SIDE];
#pragma unroll
      for (int r = 0; r < SIDE; ++r) {
        zz[r] = v[u][r] - dc;
        sq = fma(zz[r], zz[r], sq);
      }
      // rows r, r + 1 leave as 16-byte (Z64) / 8-byte (Z32) pairs: the even
      // lane of a column pair writes row r's two columns, the odd lane row
      // r + 1's, after one exchange of the element the other needs
      const bool odd = c & 1;
#pragma unroll
      for (int r = 0; r < SIDE; r += 2) {
        const double got = __shfl_xor_sync(0xffffffffu, odd ? zz[r] : zz[r + 1], 1);
        if (valid) {
          const int e = odd ? (r + 1) * SIDE + c - 1 : r * SIDE + c;
          const double a0 = odd ? got : zz[r], a1 = odd ? zz[r + 1] : got;
          if (Z64) *reinterpret_cast<double2*>(Z64 + g[u] * P + e) = make_double2(a0, a1);
          if (Z32) *reinterpret_cast<float2*>(Z32 + g[u] * z32_pitch + e) = make_float2((float)a0, (float)a1);
        }
      }
      if (valid && Z32)
        for (int p = P + c; p < z32_pitch; p += SIDE) Z32[g[u] * z32_pitch + p] = 0.0f;
#pragma unroll
      for (int h = SIDE / 2; h >= 1; h >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, h, SIDE);
      if (valid && c == 0) {
        if (dc_out) dc_out[g[u]] = dc;
        if (sq_out) sq_out[g[u]] = sq;
      }
    }
  }
}

}  // namespace fepll

// The column kernel stores rows in 16-byte (Z64) and 8-byte (Z32) pairs:
// it needs 16-byte aligned Z64, 8-byte aligned Z32 and an even z32_pitch.
// Other layouts (valid under the ABI) take the per-row-store kernel.
static bool paired_stores_ok(const double* Z64, const float* Z32, int z32_pitch) {
  return (reinterpret_cast<uintptr_t>(Z64) % 16 == 0) &&
         (Z32 == nullptr || (reinterpret_cast<uintptr_t>(Z32) % 8 == 0 && z32_pitch % 2 == 0));
}

extern "C" int fepll_extract(const double* x, int32_t batch, int32_t H, int32_t W, int32_t side,
                             const int32_t* anchors, int32_t n, int32_t grid_cols, double* Z64,
                             float* Z32, int32_t z32_pitch, double* dc, double* sq, void* stream) {
  using namespace fepll;
  FEPLL_REQUIRE(x && anchors && batch >= 1 && n >= 0, "extract: bad arguments");
  FEPLL_REQUIRE(side >= 1 && side * side <= kMaxP, "extract: patch side out of range");
  FEPLL_REQUIRE(H >= side && W >= side, "extract: image smaller than the patch");
  FEPLL_REQUIRE(Z32 == nullptr || z32_pitch >= side * side, "extract: Z32 pitch below P");
  (void)grid_cols;
  if (n == 0) return kOk;
  const int64_t total = (int64_t)batch * n;
  cudaStream_t st = (cudaStream_t)stream;
  const bool pow2 = side == 8 || side == 4 || side == 16;
  if (pow2 && paired_stores_ok(Z64, Z32, z32_pitch)) {
    const int per_warp = 32 / side;
    const int64_t warps = (total + per_warp - 1) / per_warp;
    // one lane group per warp pass (side 4: two): with the paired row stores
    // it measured 2-4 % faster than two or four (fewer registers)
    const int u = side == 4 ? 2 : 1;
    const int grid = grid_for((warps + u - 1) / u, 8, 148 * 8);
    // FP32 rows only (fp32-state): six CTAs per SM at 40 registers hide more of
    // the window-load latency (2.48 -> 2.37 ms/step at 64 x 1024^2); with the
    // FP64 rows as well the same cap measured slower (3.24 -> 3.64)
    if (side == 8 && Z64 == nullptr)
      extract_cols_kernel<8, 1, 6><<<grid_for(warps, 8, 148 * 12), 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
    else if (side == 8)
      extract_cols_kernel<8, 1><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
    else if (side == 4)
      extract_cols_kernel<4, 2><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
    else
      extract_cols_kernel<16, 1><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq);
  } else if (pow2) {
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
