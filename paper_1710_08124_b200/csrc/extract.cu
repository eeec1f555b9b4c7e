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
// same image rows, so the loads mostly hit L1).  The fold is the tile
// kernel's (row halvings in registers, column halvings by shuffles: the same
// FP64 additions as patches.py:153-164), and every row of Z64 / Z32 leaves as
// one SIDE-lane store (64 B / 32 B segments per patch row at SIDE = 8).  No
// shared memory, no barriers: a few dozen instructions per patch, where the
// staged tile kernel spends several hundred on its staging loops.
template <int SIDE, int U>
__global__ void __launch_bounds__(256)
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

int g_extract_variant = 0;  // debug: 1 = staged tile kernel, 2 = U=2, 4 = U=4

// Tiled variant for power-of-two sides on a row-major anchor grid: a block
// takes PB consecutive anchors of one nominal row (grid_cols anchors per
// row), stages the image window they touch in shared memory with coalesced
// loads, runs the same shuffle fold per patch (bitwise-equal dc), stages the
// patch rows, and writes the block's contiguous Z64 / Z32 span with 16-byte
// stores — the per-lane 8-byte global accesses of extract_pow2_kernel were
// LSU-issue bound.  Blocks whose window exceeds the staging area (irregular
// anchors) read the image directly.
template <int SIDE>
__global__ void __launch_bounds__(256)
extract_tile_kernel(const double* __restrict__ x, int batch, int H, int W,
                    const int32_t* __restrict__ anchors, int n, int grid_cols, int win_cap,
                    double* __restrict__ Z64, float* __restrict__ Z32, int z32_pitch,
                    double* __restrict__ dc_out, double* __restrict__ sq_out) {
  constexpr int P = SIDE * SIDE;
  constexpr int PER_WARP = 32 / SIDE;
  constexpr int PB = 8 * PER_WARP;  // patches per block
  extern __shared__ __align__(16) double sm[];
  double* zs = sm;                       // [PB][P] staged FP64 rows
  double* win = sm + PB * P;             // [rows][cols] image window (win_cap doubles)
  __shared__ int s_pr[PB], s_pc[PB];
  __shared__ int s_lo[2], s_hi[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col_blocks = (grid_cols + PB - 1) / PB;
  const int rows_total = n / grid_cols;
  for (int64_t blk = blockIdx.x; blk < (int64_t)batch * rows_total * col_blocks; blk += gridDim.x) {
    const int b = (int)(blk / ((int64_t)rows_total * col_blocks));
    const int rem = (int)(blk - (int64_t)b * rows_total * col_blocks);
    const int a = rem / col_blocks, cb = rem - a * col_blocks;
    const int i0 = a * grid_cols + cb * PB;
    const int m = min(PB, grid_cols - cb * PB);
    const int64_t g0 = (int64_t)b * n + i0;
    if (tid < 2) {
      s_lo[tid] = INT_MAX;
      s_hi[tid] = INT_MIN;
    }
    __syncthreads();
    if (tid < m) {
      const int pr = anchors[2 * (i0 + tid)], pc = anchors[2 * (i0 + tid) + 1];
      s_pr[tid] = pr;
      s_pc[tid] = pc;
      atomicMin(&s_lo[0], pr);
      atomicMax(&s_hi[0], pr);
      atomicMin(&s_lo[1], pc);
      atomicMax(&s_hi[1], pc);
    }
    __syncthreads();
    const int r_lo = s_lo[0], c_lo = s_lo[1];
    const int wr = s_hi[0] - r_lo + SIDE, wc = s_hi[1] - c_lo + SIDE;
    const bool staged = wr * wc <= win_cap;
    const double* img = x + (int64_t)b * H * W;
    if (staged) {
      for (int r = warp; r < wr; r += 8) {
        const double* src = img + (int64_t)(r_lo + r) * W + c_lo;
        for (int c = lane; c < wc; c += 32) win[r * wc + c] = __ldg(src + c);
      }
    }
    __syncthreads();
    // one lane group per patch, lane c = window COLUMN c: the reference's
    // halvings of the flattened row (patches.py:156-163) first add row r + h
    // to row r elementwise — in-register adds down this lane's column — and
    // then halve the surviving row across the group's lanes: the same FP64
    // additions in the same order as extract_pow2_kernel, a fraction of its
    // shuffles
    const int p = warp * PER_WARP + lane / SIDE;
    const int c = lane % SIDE;
    const bool valid = p < m;
    double v[SIDE];  // v[r] = window(r, c)
    if (valid) {
      const int pr = s_pr[p], pc = s_pc[p];
      if (staged) {
        const double* src = win + (pr - r_lo) * wc + (pc - c_lo + c);
#pragma unroll
        for (int r = 0; r < SIDE; ++r) v[r] = src[r * wc];
      } else {
        const double* src = img + (int64_t)pr * W + pc + c;
#pragma unroll
        for (int r = 0; r < SIDE; ++r) v[r] = __ldg(src + (int64_t)r * W);
      }
    } else {
#pragma unroll
      for (int r = 0; r < SIDE; ++r) v[r] = 0.0;
    }
    double acc[SIDE];
#pragma unroll
    for (int r = 0; r < SIDE; ++r) acc[r] = v[r];
#pragma unroll
    for (int h = SIDE / 2; h >= 1; h >>= 1)
#pragma unroll
      for (int r = 0; r < h; ++r) acc[r] = acc[r] + acc[r + h];
    double col = acc[0];  // row 0 of the halved rows, column c
#pragma unroll
    for (int h = SIDE / 2; h >= 1; h >>= 1) {
      const double o = __shfl_down_sync(0xffffffffu, col, h, SIDE);
      if (c < h) col = col + o;
    }
    const double dc = __shfl_sync(0xffffffffu, col, 0, SIDE) / (double)P;
    double sq = 0.0;
    if (valid) {
      double* zcol = zs + p * P + c;
#pragma unroll
      for (int r = 0; r < SIDE; ++r) {
        const double z = v[r] - dc;
        sq = fma(z, z, sq);
        zcol[r * SIDE] = z;
      }
    }
#pragma unroll
    for (int h = SIDE / 2; h >= 1; h >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, h, SIDE);
    if (valid && c == 0) {
      if (dc_out) dc_out[g0 + p] = dc;
      if (sq_out) sq_out[g0 + p] = sq;
    }
    __syncthreads();
    // contiguous spans: m rows of Z64 (P doubles), m rows of Z32 (z32_pitch floats)
    if (Z64) {
      const double2* src = reinterpret_cast<const double2*>(zs);
      double2* dst = reinterpret_cast<double2*>(Z64 + g0 * P);
      for (int k = tid; k < m * P / 2; k += 256) dst[k] = src[k];
    }
    if (Z32 && z32_pitch == P) {  // no padding: a flat conversion
      const double2* src = reinterpret_cast<const double2*>(zs);
      float4* dst = reinterpret_cast<float4*>(Z32 + g0 * P);
      for (int k = tid; k < m * P / 4; k += 256) {
        const double2 a0 = src[2 * k], a1 = src[2 * k + 1];
        dst[k] = make_float4((float)a0.x, (float)a0.y, (float)a1.x, (float)a1.y);
      }
    } else if (Z32) {
      const int q4 = z32_pitch / 4;
      float4* dst = reinterpret_cast<float4*>(Z32 + g0 * z32_pitch);
      for (int k = tid; k < m * q4; k += 256) {
        const int row = k / q4, col = (k - row * q4) * 4;
        float4 f;
        f.x = col + 0 < P ? (float)zs[row * P + col + 0] : 0.0f;
        f.y = col + 1 < P ? (float)zs[row * P + col + 1] : 0.0f;
        f.z = col + 2 < P ? (float)zs[row * P + col + 2] : 0.0f;
        f.w = col + 3 < P ? (float)zs[row * P + col + 3] : 0.0f;
        dst[k] = f;
      }
    }
    __syncthreads();
  }
}

template <int SIDE>
static void launch_tile(const double* x, int batch, int H, int W, const int32_t* anchors, int n,
                        int grid_cols, double* Z64, float* Z32, int z32_pitch, double* dc, double* sq,
                        cudaStream_t st) {
  constexpr int P = SIDE * SIDE;
  constexpr int PB = 8 * (32 / SIDE);
  const int win_cap = SIDE == 16 ? 8192 : 2048;  // staged window (doubles)
  const size_t smem = sizeof(double) * ((size_t)PB * P + win_cap);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(extract_tile_kernel<SIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t blocks = (int64_t)batch * (n / grid_cols) * ((grid_cols + PB - 1) / PB);
  extract_tile_kernel<SIDE><<<grid_for(blocks, 1, kSMs * 8), 256, smem, st>>>(
      x, batch, H, W, anchors, n, grid_cols, win_cap, Z64, Z32, z32_pitch, dc, sq);
}

}  // namespace fepll

extern "C" int fepll_extract(const double* x, int32_t batch, int32_t H, int32_t W, int32_t side,
                             const int32_t* anchors, int32_t n, int32_t grid_cols, double* Z64,
                             float* Z32, int32_t z32_pitch, double* dc, double* sq, void* stream) {
  using namespace fepll;
  FEPLL_REQUIRE(x && anchors && batch >= 1 && n >= 0, "extract: bad arguments");
  FEPLL_REQUIRE(side >= 1 && side * side <= kMaxP, "extract: patch side out of range");
  FEPLL_REQUIRE(H >= side && W >= side, "extract: image smaller than the patch");
  FEPLL_REQUIRE(Z32 == nullptr || z32_pitch >= side * side, "extract: Z32 pitch below P");
  if (n == 0) return kOk;
  const int64_t total = (int64_t)batch * n;
  cudaStream_t st = (cudaStream_t)stream;
  if (g_extract_variant != 1 && (side == 8 || side == 4 || side == 16)) {
    const int per_warp = 32 / side;
    const int64_t warps = (total + per_warp - 1) / per_warp;
    // one lane group per warp pass: with the paired row stores it measured
    // 2-4 % faster than two (fewer registers); debug 2: U=2, 4: U=4
    const int u = g_extract_variant == 0 ? 1 : g_extract_variant == 2 ? 2 : 4;
    const int grid = grid_for((warps + u - 1) / u, 8, 148 * 8);
#define FEPLL_EXT(S, U) extract_cols_kernel<S, U><<<grid, 256, 0, st>>>(x, batch, H, W, anchors, n, Z64, Z32, z32_pitch, dc, sq)
    if (side == 8) {
      if (u == 1) FEPLL_EXT(8, 1); else if (u == 2) FEPLL_EXT(8, 2); else FEPLL_EXT(8, 4);
    } else if (side == 4) {
      FEPLL_EXT(4, 2);
    } else {
      FEPLL_EXT(16, 1);
    }
#undef FEPLL_EXT
  } else if (grid_cols > 0 && n % grid_cols == 0 && (side == 8 || side == 4 || side == 16) &&
      (Z32 == nullptr || z32_pitch % 4 == 0)) {
    if (side == 8)
      launch_tile<8>(x, batch, H, W, anchors, n, grid_cols, Z64, Z32, z32_pitch, dc, sq, st);
    else if (side == 4)
      launch_tile<4>(x, batch, H, W, anchors, n, grid_cols, Z64, Z32, z32_pitch, dc, sq, st);
    else
      launch_tile<16>(x, batch, H, W, anchors, n, grid_cols, Z64, Z32, z32_pitch, dc, sq, st);
  } else if (side == 8 || side == 4 || side == 16) {
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

extern "C" int fepll_debug_extract_variant(int32_t v) {
  fepll::g_extract_variant = v;
  return 0;
}
