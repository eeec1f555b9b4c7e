// Is mma.sync m16n8k8.f64 bitwise the same as two m8n8k4.f64 steps (k 0-3,
// then k 4-7) per 8-row half, and as a sequential FMA chain over k?  (Decides
// whether the Wiener kernel may switch DMMA shapes without changing a bit.)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dmma_order_probe.cu -o tools/dmma_order_probe
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

__device__ __forceinline__ void m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void m16n8k8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// A: [trials][16][8] row-major, B: [trials][8][8] (k x n), C0: [trials][16][8] initial
__global__ void probe(const double* A, const double* B, const double* C0, double* D16, double* D8, int trials) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  for (int tr = blockIdx.x; tr < trials; tr += gridDim.x) {
    const double* a = A + tr * 128;
    const double* b = B + tr * 64;
    const double* c = C0 + tr * 128;
    double d[4] = {c[g * 8 + 2 * t], c[g * 8 + 2 * t + 1], c[(g + 8) * 8 + 2 * t], c[(g + 8) * 8 + 2 * t + 1]};
    double e[4] = {d[0], d[1], d[2], d[3]};
    const double af[4] = {a[g * 8 + t], a[(g + 8) * 8 + t], a[g * 8 + t + 4], a[(g + 8) * 8 + t + 4]};
    const double bf[2] = {b[t * 8 + g], b[(t + 4) * 8 + g]};
    m16n8k8(d, af, bf);
    m8n8k4(e[0], e[1], af[0], bf[0]);
    m8n8k4(e[2], e[3], af[1], bf[0]);
    m8n8k4(e[0], e[1], af[2], bf[1]);
    m8n8k4(e[2], e[3], af[3], bf[1]);
    double* o16 = D16 + tr * 128;
    double* o8 = D8 + tr * 128;
    o16[g * 8 + 2 * t] = d[0]; o16[g * 8 + 2 * t + 1] = d[1];
    o16[(g + 8) * 8 + 2 * t] = d[2]; o16[(g + 8) * 8 + 2 * t + 1] = d[3];
    o8[g * 8 + 2 * t] = e[0]; o8[g * 8 + 2 * t + 1] = e[1];
    o8[(g + 8) * 8 + 2 * t] = e[2]; o8[(g + 8) * 8 + 2 * t + 1] = e[3];
  }
}

int main() {
  const int trials = 20000;
  std::vector<double> A(trials * 128), B(trials * 64), C(trials * 128);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::uniform_int_distribution<int> ex(-30, 30);
  for (auto& v : A) v = std::ldexp(nd(rng), ex(rng) / 3);
  for (auto& v : B) v = std::ldexp(nd(rng), ex(rng) / 3);
  for (auto& v : C) v = std::ldexp(nd(rng), ex(rng));
  double *dA, *dB, *dC, *d16, *d8;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
  cudaMalloc(&d16, C.size() * 8); cudaMalloc(&d8, C.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  probe<<<148, 32>>>(dA, dB, dC, d16, d8, trials);
  std::vector<double> o16(C.size()), o8(C.size());
  cudaMemcpy(o16.data(), d16, C.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(o8.data(), d8, C.size() * 8, cudaMemcpyDeviceToHost);
  long diff_16_8 = 0, diff_8_fma = 0, diff_16_fma = 0;
  for (int tr = 0; tr < trials; ++tr)
    for (int m = 0; m < 16; ++m)
      for (int n = 0; n < 8; ++n) {
        const int i = tr * 128 + m * 8 + n;
        double s = C[i];
        for (int k = 0; k < 8; ++k) s = std::fma(A[tr * 128 + m * 8 + k], B[tr * 64 + k * 8 + n], s);
        if (std::memcmp(&o16[i], &o8[i], 8)) ++diff_16_8;
        if (std::memcmp(&o8[i], &s, 8)) ++diff_8_fma;
        if (std::memcmp(&o16[i], &s, 8)) ++diff_16_fma;
      }
  printf("elements %d: m16n8k8 != 2 x m8n8k4: %ld; m8n8k4 != sequential fma: %ld; m16n8k8 != sequential fma: %ld (%s)\n",
         trials * 128, diff_16_8, diff_8_fma, diff_16_fma, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
