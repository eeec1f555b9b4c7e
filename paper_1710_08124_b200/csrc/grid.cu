// Sampling plans on the device: the jittered anchor grid of
// pkg/src/fepll/patches.py:102-132 (and the regular grid of :89-99),
// bit-identical to numpy's Generator(Philox(key=[seed, t])).integers stream.
//
// The stream is counter-indexed: uint32 draw j is half (j & 1: high) of
// word (j/2) % 4 of Philox4x64-10 block j/8, computed with counter
// [j/8 + 1, 0, 0, 0] (numpy bumps the counter before each block) — so any
// thread can produce any draw.  Generator.integers over a range of n values
// is Lemire's multiply with rejection: draw u is accepted iff
// (u*n mod 2^32) >= (2^32 - n) mod n and maps to (u*n) >> 32; rejected draws
// are skipped.  Rejections are rare (n / 2^32 per draw), so the generator
// (1) draws the two global-shift values serially, (2) flags the rejected
// positions of the jitter window in parallel, (3) sorts that short list, and
// (4) emits every anchor from its stream position shifted past the rejected
// positions before it.  The 128-bit key is the one numpy derives from
// Philox(key=[seed & (2^64-1), t]) (the host passes its two words, so even
// numpy's conversion of the key list is reproduced).
// oracle/fepll_oracle.py:jittered_grid_counter is the CPU model of the same
// arithmetic, pinned to numpy.
#include "common.cuh"

namespace fepll {

namespace grid {

constexpr int kMaxRejects = 256;  // rejected draws tolerated per grid (expected: ~0)

// scratch layout (int32)
constexpr int kJ0 = 0, kShift0 = 1, kShift1 = 2, kRejects = 3, kList = 8;
constexpr int kScratchInts = kList + kMaxRejects;

struct U4 {
  uint64_t v[4];
};

__device__ __forceinline__ U4 philox4x64_10(uint64_t c0, uint64_t key0, uint64_t key1) {
  uint64_t c[4] = {c0, 0, 0, 0};
  uint64_t k0 = key0, k1 = key1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
    const uint64_t lo0 = m0 * c[0], hi0 = __umul64hi(m0, c[0]);
    const uint64_t lo1 = m1 * c[2], hi1 = __umul64hi(m1, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
  U4 o;
#pragma unroll
  for (int i = 0; i < 4; ++i) o.v[i] = c[i];
  return o;
}

__device__ __forceinline__ uint32_t draw32(uint64_t key0, uint64_t key1, int64_t j) {
  const int64_t q = j >> 1;
  const U4 b = philox4x64_10((uint64_t)(q >> 2) + 1, key0, key1);
  const uint64_t w = b.v[q & 3];
  return (j & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
}

__host__ __device__ inline uint32_t lemire_threshold(uint32_t n_excl) {
  return (uint32_t)((((uint64_t)1 << 32) - n_excl) % n_excl);
}

// axis_anchors (patches.py:79-86): k*s, the last one clamped to extent-side
__device__ __forceinline__ int axis_anchor(int k, int count, int last, int s) {
  return k == count - 1 ? last : k * s;
}

__global__ void shift_kernel(uint64_t key0, uint64_t key1, int spacing, int draw_shift, uint32_t th_override,
                             int32_t* scratch) {
  int64_t j = 0;
  int32_t shift[2] = {0, 0};
  if (draw_shift) {
    const uint32_t n = (uint32_t)spacing;
    const uint32_t th = th_override ? th_override : lemire_threshold(n);
    for (int k = 0; k < 2; ++k) {
      for (;;) {
        const uint64_t m = (uint64_t)draw32(key0, key1, j++) * n;
        if ((uint32_t)m >= th) {
          shift[k] = (int32_t)(m >> 32);
          break;
        }
      }
    }
  }
  scratch[kJ0] = (int32_t)j;
  scratch[kShift0] = shift[0];
  scratch[kShift1] = shift[1];
  scratch[kRejects] = 0;
}

// flag rejected positions of [j0, j0 + count): one thread per Philox block
__global__ void flag_kernel(uint64_t key0, uint64_t key1, int64_t count, uint32_t n_excl, uint32_t th,
                            int32_t* scratch) {
  const int64_t j0 = scratch[kJ0];
  const int64_t first_block = j0 >> 3;
  const int64_t last_block = (j0 + count - 1) >> 3;
  for (int64_t b = first_block + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= last_block;
       b += (int64_t)gridDim.x * blockDim.x) {
    const U4 w = philox4x64_10((uint64_t)b + 1, key0, key1);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int64_t j = b * 8 + h;
      if (j < j0 || j >= j0 + count) continue;
      const uint32_t u = (h & 1) ? (uint32_t)(w.v[h >> 1] >> 32) : (uint32_t)w.v[h >> 1];
      const uint64_t m = (uint64_t)u * n_excl;
      if ((uint32_t)m < th) {
        const int idx = atomicAdd(&scratch[kRejects], 1);
        if (idx < kMaxRejects) scratch[kList + idx] = (int32_t)j;
      }
    }
  }
}

__global__ void sort_kernel(int32_t* scratch, int32_t* status) {
  const int r = scratch[kRejects];
  if (r >= kMaxRejects) {
    atomicOr(status, 4);
    return;
  }
  int32_t* l = scratch + kList;
  for (int i = 1; i < r; ++i) {
    const int32_t v = l[i];
    int k = i - 1;
    while (k >= 0 && l[k] > v) {
      l[k + 1] = l[k];
      --k;
    }
    l[k + 1] = v;
  }
}

// number of listed rejections <= pos
__device__ __forceinline__ int rejects_upto(const int32_t* l, int r, int64_t pos) {
  int lo = 0, hi = r;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (l[mid] <= pos) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void emit_kernel(uint64_t key0, uint64_t key1, int H, int W, int side, int spacing, int half,
                            int n_rows, int n_cols, int jitter, uint32_t n_excl,
                            const int32_t* __restrict__ scratch, int32_t* __restrict__ anchors) {
  __shared__ int32_t l[kMaxRejects];
  const int r = jitter ? min(scratch[kRejects], kMaxRejects) : 0;
  for (int i = threadIdx.x; i < r; i += blockDim.x) l[i] = scratch[kList + i];
  __syncthreads();
  const int64_t n = (int64_t)n_rows * n_cols;
  const int last_r = H - side, last_c = W - side;
  const int64_t j0 = jitter ? scratch[kJ0] : 0;
  const int band0 = jitter ? scratch[kShift0] % (2 * half + 1) - half : 0;
  const int band1 = jitter ? scratch[kShift1] % (2 * half + 1) - half : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ia = (int)(i / n_cols), ib = (int)(i - (int64_t)ia * n_cols);
    const int R = axis_anchor(ia, n_rows, last_r, spacing);
    const int Cc = axis_anchor(ib, n_cols, last_c, spacing);
    int pr = R, pc = Cc;
    if (jitter) {
      int off[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        // stream position of output 2i + a, skipping listed rejections
        const int64_t base = j0 + 2 * i + a;
        int k = 0;
        for (;;) {
          const int k2 = rejects_upto(l, r, base + k);
          if (k2 == k) break;
          k = k2;
        }
        const uint64_t m = (uint64_t)draw32(key0, key1, base + k) * n_excl;
        const int jit = (int)(m >> 32) - half;
        const int o = min(max((a ? band1 : band0) + jit, -half), half);
        off[a] = o;
      }
      if (R == 0 || R == last_r) off[0] = 0;
      if (Cc == 0 || Cc == last_c) off[1] = 0;
      pr = min(max(R + off[0], 0), last_r);
      pc = min(max(Cc + off[1], 0), last_c);
    }
    anchors[2 * i] = pr;
    anchors[2 * i + 1] = pc;
  }
}

static int axis_count(int extent, int side, int s) {
  const int last = extent - side;
  return last / s + 1 + (last % s != 0 ? 1 : 0);
}

}  // namespace grid

}  // namespace fepll

extern "C" int fepll_grid_scratch_ints(void) { return fepll::grid::kScratchInts; }

extern "C" int fepll_sample_grid(uint64_t key0, uint64_t key1, int32_t H, int32_t W, int32_t side,
                                 int32_t spacing, int32_t jittered, uint32_t threshold_override,
                                 int32_t* anchors, int32_t* scratch, int32_t* status, void* stream) {
  using namespace fepll;
  using namespace fepll::grid;
  FEPLL_REQUIRE(anchors && scratch && status, "sample_grid: bad arguments");
  FEPLL_REQUIRE(side >= 1 && spacing >= 1 && spacing <= side, "sample_grid: spacing must lie in [1, side]");
  FEPLL_REQUIRE(H >= side && W >= side, "sample_grid: image smaller than the patch");
  cudaStream_t st = (cudaStream_t)stream;
  const int n_rows = axis_count(H, side, spacing), n_cols = axis_count(W, side, spacing);
  const int64_t n = (int64_t)n_rows * n_cols;
  const int half = (side - spacing) / 2;
  const int jitter = jittered && half > 0;
  const uint32_t n_excl = 2u * half + 1u;
  if (jitter) {
    shift_kernel<<<1, 1, 0, st>>>(key0, key1, spacing, spacing > 1, threshold_override, scratch);
    FEPLL_LAUNCH();
    const int64_t count = 2 * n + kMaxRejects;
    const uint32_t th = threshold_override ? threshold_override : lemire_threshold(n_excl);
    flag_kernel<<<grid_for((count + 7) / 8 + 1, 256, kSMs * 8), 256, 0, st>>>(key0, key1, count,
                                                                            n_excl, th, scratch);
    FEPLL_LAUNCH();
    sort_kernel<<<1, 1, 0, st>>>(scratch, status);
    FEPLL_LAUNCH();
  }
  emit_kernel<<<grid_for(n, 256, kSMs * 8), 256, 0, st>>>(key0, key1, H, W, side, spacing, half,
                                                         n_rows, n_cols, jitter, n_excl, scratch, anchors);
  FEPLL_LAUNCH();
  return kOk;
}
