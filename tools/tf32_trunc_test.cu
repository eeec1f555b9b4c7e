// Does tcgen05 kind::tf32 truncate or round FP32 operands that are not
// TF32-representable?  A (128 x 32, random FP32) times B (16 x 32, small
// integers, exact in TF32); compare D with host products of trunc(A) and
// rna(A).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1710_08124_b200/csrc tools/tf32_trunc_test.cu -o tools/tf32_trunc_test
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include "tc.cuh"

using namespace fepll;

__global__ void k(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[16 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem;
  const int tid = threadIdx.x;
  // swizzled K-major: row r, 16-byte chunk c at (r/8)*1024 + (r%8)*128 + ((c ^ r%8) * 16)
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int r = e / 8, c = e % 8;
    *reinterpret_cast<float4*>(sa + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) << 4)) =
        *reinterpret_cast<const float4*>(A + r * 32 + c * 4);
  }
  for (int e = tid; e < 16 * 8; e += blockDim.x) {
    const int r = e / 8, c = e % 8;
    *reinterpret_cast<float4*>(sb + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) << 4)) =
        *reinterpret_cast<const float4*>(B + r * 32 + c * 4);
  }
  tc::fence_proxy_async_smem();
  if (tid < 32) tc::tmem_alloc(&tmem, 32);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, 16);
    for (int kk = 0; kk < 4; ++kk)
      tc::mma_tf32(tmem, tc::desc_sw128(tc::smem_u32(sa) + kk * 32), tc::desc_sw128(tc::smem_u32(sb) + kk * 32),
                   idesc, kk > 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  const int warp = tid / 32, lane = tid % 32;
  uint32_t r[32];
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
  tc::tmem_ld_wait();
  for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 16 + j] = __uint_as_float(r[j]);
  tc::fence_before_sync();
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(tmem, 32);
}

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
static float rna_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  std::mt19937 g(3);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> A(128 * 32), B(16 * 32), D(128 * 16);
  for (auto& v : A) v = U(g);
  for (int i = 0; i < 16 * 32; ++i) B[i] = (float)((int)(g() % 9) - 4);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dA, dB, dD);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double et = 0, er = 0, ex = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      double st = 0, sr = 0, sx = 0;
      for (int k2 = 0; k2 < 32; ++k2) {
        st += (double)trunc_tf32(A[m * 32 + k2]) * B[n * 32 + k2];
        sr += (double)rna_tf32(A[m * 32 + k2]) * B[n * 32 + k2];
        sx += (double)A[m * 32 + k2] * B[n * 32 + k2];
      }
      const double d = D[m * 16 + n];
      et = fmax(et, fabs(d - st)); er = fmax(er, fabs(d - sr)); ex = fmax(ex, fabs(d - sx));
    }
  printf("max |D - trunc| %.3g   |D - rna| %.3g   |D - fp32 exact| %.3g\n", et, er, ex);
  return 0;
}
