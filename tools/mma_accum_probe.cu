// Probe of the FP32 accumulation inside tcgen05 kind::tf32 and kind::f16
// (bf16) MMAs — the hardware behaviour the certified argmin's error budget
// (csrc/select_ws2.cu header, csrc/tc_epi.cuh) rests on.
//
// The budget assumes each output element of the ws2 tree-level kernel — 8
// kind::tf32 MMAs (K = 64) followed by 8 kind::f16 MMAs (bf16, K = 128) into
// one FP32 accumulator — is within 16 * 2^-23 * sum_k |a_k b_k| of the exact
// sum of the products of the operands as the hardware reads them (tf32:
// truncated FP32, tools/tf32_trunc_test.cu; bf16: exact).  That is one FP32
// rounding (round-to-zero allowed: one ulp, not half) per MMA step.
//
// For several adversarial input families this measures, per mode,
//   max |D - exact| / sum_k |a_k b_k|   in units of 2^-23,
// and whether D equals the sequentially round-to-nearest FP32 result.  The
// program exits 1 if any mode exceeds its budget (8 units for the single
// passes, 16 for the combined ws2 pattern).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//      -I paper_1710_08124_b200/csrc tools/mma_accum_probe.cu -o tools/mma_accum_probe
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "tc.cuh"

using namespace fepll;

constexpr int kM = 128, kN = 16;
constexpr int kK32 = 64;   // tf32 pass: 8 MMAs of K = 8
constexpr int kK16 = 128;  // bf16 pass: 8 MMAs of K = 16

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc) : "memory");
}

// rows x 256-byte K-major matrix -> SWIZZLE_128B image: two 128-byte K atoms,
// atom ka at ka * rows * 128 bytes, row r's 16-byte chunk c at
// (r / 8) * 1024 + (r % 8) * 128 + ((c ^ r % 8) * 16)
__device__ void stage(uint8_t* dst, const uint8_t* src, int rows) {
  for (int e = threadIdx.x; e < rows * 16; e += blockDim.x) {
    const int r = e / 16, c16 = e % 16, ka = c16 / 8, c = c16 % 8;
    *reinterpret_cast<uint4*>(dst + ka * rows * 128 + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) << 4)) =
        *reinterpret_cast<const uint4*>(src + (size_t)r * 256 + c16 * 16);
  }
}

// mode 0: tf32 pass only, 1: bf16 pass only, 2: tf32 then bf16 (ws2 pattern)
__global__ void probe(int mode, const float* A32, const float* B32, const uint16_t* A16, const uint16_t* B16,
                      float* D) {
  extern __shared__ uint8_t dyn[];
  uint8_t* base = tc::align1024(dyn);
  uint8_t* sa32 = base;                 // 32 KB
  uint8_t* sb32 = base + 32768;         // 4 KB
  uint8_t* sa16 = base + 32768 + 4096;  // 32 KB
  uint8_t* sb16 = sa16 + 32768;         // 4 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem;
  const size_t cta = blockIdx.x;
  stage(sa32, reinterpret_cast<const uint8_t*>(A32 + cta * kM * kK32), kM);
  stage(sb32, reinterpret_cast<const uint8_t*>(B32 + cta * kN * kK32), kN);
  stage(sa16, reinterpret_cast<const uint8_t*>(A16 + cta * kM * kK16), kM);
  stage(sb16, reinterpret_cast<const uint8_t*>(B16 + cta * kN * kK16), kN);
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc(&tmem, 32);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x == 0) {
    int acc = 0;
    if (mode != 1) {
      const uint32_t id = tc::idesc_tf32(kM, kN);
      for (int kk = 0; kk < 8; ++kk, acc = 1)
        tc::mma_tf32(tmem, tc::desc_sw128(tc::smem_u32(sa32) + (kk / 4) * kM * 128 + (kk % 4) * 32),
                     tc::desc_sw128(tc::smem_u32(sb32) + (kk / 4) * kN * 128 + (kk % 4) * 32), id, acc);
    }
    if (mode != 0) {
      const uint32_t id = tc::idesc_bf16(kM, kN);
      for (int kk = 0; kk < 8; ++kk, acc = 1)
        mma_f16_ss(tmem, tc::desc_sw128(tc::smem_u32(sa16) + (kk / 4) * kM * 128 + (kk % 4) * 32),
                   tc::desc_sw128(tc::smem_u32(sb16) + (kk / 4) * kN * 128 + (kk % 4) * 32), id, acc);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t r[32];
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
  tc::tmem_ld_wait();
  for (int j = 0; j < kN; ++j) D[(cta * kM + warp * 32 + lane) * kN + j] = __uint_as_float(r[j]);
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 32);
}

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
static uint16_t bf16_rne(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
static float bf16_val(uint16_t h) { uint32_t u = (uint32_t)h << 16; float y; memcpy(&y, &u, 4); return y; }

// one input family: fills one CTA's operands
struct Family {
  const char* name;
  int id;
};

static float draw(std::mt19937_64& g, int fam, int k, int K) {
  std::uniform_real_distribution<double> U(-1.0, 1.0), E(-24.0, 0.0);
  switch (fam) {
    case 0: return (float)U(g);                                         // uniform
    case 1: return (float)(std::copysign(std::exp2(E(g)), U(g)));      // spread exponents
    case 2: return k == 0 ? 1.0f : (float)(U(g) * std::exp2(-13.0));   // one big + many small
    case 3: return (float)((k & 1 ? -1.0 : 1.0) * (1.0 + std::ldexp(U(g), -8)));  // alternating cancellation
    default: return (float)(U(g) * std::exp2((double)(k % 9) * -3.0)); // staircase magnitudes
  }
}

int main() {
  const int ctas = 148, fams = 5;
  const size_t na32 = (size_t)ctas * kM * kK32, nb32 = (size_t)ctas * kN * kK32;
  const size_t na16 = (size_t)ctas * kM * kK16, nb16 = (size_t)ctas * kN * kK16;
  float *dA32, *dB32, *dD;
  uint16_t *dA16, *dB16;
  cudaMalloc(&dA32, na32 * 4); cudaMalloc(&dB32, nb32 * 4);
  cudaMalloc(&dA16, na16 * 2); cudaMalloc(&dB16, nb16 * 2);
  cudaMalloc(&dD, (size_t)ctas * kM * kN * 4);
  const int smem = 32768 * 2 + 4096 * 2 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* fam_name[fams] = {"uniform", "spread-exp", "big+small", "cancel", "staircase"};
  const char* mode_name[3] = {"tf32 x8 (K=64)", "bf16 x8 (K=128)", "tf32 x8 + bf16 x8 (ws2)"};
  const double budget[3] = {8.0, 8.0, 16.0};
  bool ok = true;
  std::mt19937_64 g(12345);
  std::vector<float> A32(na32), B32(nb32), D((size_t)ctas * kM * kN);
  std::vector<uint16_t> A16(na16), B16(nb16);
  for (int mode = 0; mode < 3; ++mode) {
    double worst_all = 0.0;
    for (int fam = 0; fam < fams; ++fam) {
      for (size_t i = 0; i < na32; ++i) A32[i] = draw(g, fam, (int)(i % kK32), kK32);
      for (size_t i = 0; i < nb32; ++i) B32[i] = draw(g, fam == 3 ? 0 : fam, (int)(i % kK32), kK32);
      for (size_t i = 0; i < na16; ++i) A16[i] = bf16_rne(draw(g, fam, (int)(i % kK16), kK16));
      for (size_t i = 0; i < nb16; ++i) B16[i] = bf16_rne(draw(g, fam == 3 ? 0 : fam, (int)(i % kK16), kK16));
      cudaMemcpy(dA32, A32.data(), na32 * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dB32, B32.data(), nb32 * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dA16, A16.data(), na16 * 2, cudaMemcpyHostToDevice);
      cudaMemcpy(dB16, B16.data(), nb16 * 2, cudaMemcpyHostToDevice);
      probe<<<ctas, 128, smem>>>(mode, dA32, dB32, dA16, dB16, dD);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("kernel: %s\n", cudaGetErrorString(e)); return 2; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double worst = 0.0;
      long eq_seq = 0, total = 0, below = 0, above = 0;
      for (int c = 0; c < ctas; ++c)
        for (int m = 0; m < kM; ++m)
          for (int n = 0; n < kN; ++n) {
            double ex = 0.0, mag = 0.0;
            float seq = 0.0f;
            if (mode != 1)
              for (int k = 0; k < kK32; ++k) {
                const double p = (double)trunc_tf32(A32[((size_t)c * kM + m) * kK32 + k]) *
                                 (double)trunc_tf32(B32[((size_t)c * kN + n) * kK32 + k]);
                ex += p; mag += std::fabs(p); seq += (float)p;
              }
            if (mode != 0)
              for (int k = 0; k < kK16; ++k) {
                const double p = (double)bf16_val(A16[((size_t)c * kM + m) * kK16 + k]) *
                                 (double)bf16_val(B16[((size_t)c * kN + n) * kK16 + k]);
                ex += p; mag += std::fabs(p); seq += (float)p;
              }
            const double d = D[((size_t)c * kM + m) * kN + n];
            if (mag > 0) worst = std::fmax(worst, std::fabs(d - ex) / mag / std::ldexp(1.0, -23));
            eq_seq += d == (double)seq;
            below += std::fabs(d) < std::fabs(ex);
            above += std::fabs(d) > std::fabs(ex);
            ++total;
          }
      printf("%-26s %-11s max err %6.3f x 2^-23 sum|ab|   |D|<|exact| %5.1f%%  |D|>|exact| %5.1f%%  "
             "D == sequential RN fp32 %5.1f%%\n",
             mode_name[mode], fam_name[fam], worst, 100.0 * below / total, 100.0 * above / total,
             100.0 * eq_seq / total);
      worst_all = std::fmax(worst_all, worst);
    }
    const bool pass = worst_all <= budget[mode];
    ok = ok && pass;
    printf("%-26s worst %.3f x 2^-23 vs budget %.0f: %s\n\n", mode_name[mode], worst_all, budget[mode],
           pass ? "within" : "EXCEEDED");
  }
  printf("%s\n", ok ? "PASS: the certification budget holds" : "FAIL");
  return ok ? 0 : 1;
}
