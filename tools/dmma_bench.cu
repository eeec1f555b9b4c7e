// FP64 mma.sync shapes on sm_100a: fragment-layout check against a host
// product and issue throughput (cycles per instruction per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dmma_bench.cu -o tools/dmma_bench
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>

__device__ __forceinline__ void m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void m16n8k4(double (&d)[4], const double (&a)[2], double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void m16n8k8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void m16n8k16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// A: 16 x 16 row-major, B: 16 x 8 (k x n) row-major; D = A[:, :K] B[:K, :]
__global__ void layout_check(const double* A, const double* B, double* D, int shape) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double d[4] = {0, 0, 0, 0};
  if (shape == 1) {
    double a[2] = {A[g * 16 + t], A[(g + 8) * 16 + t]};
    m16n8k4(d, a, B[t * 8 + g]);
  } else if (shape == 2) {
    double a[4] = {A[g * 16 + t], A[(g + 8) * 16 + t], A[g * 16 + t + 4], A[(g + 8) * 16 + t + 4]};
    double b[2] = {B[t * 8 + g], B[(t + 4) * 8 + g]};
    m16n8k8(d, a, b);
  } else {
    double a[8], b[4];
    for (int i = 0; i < 4; ++i) {
      a[2 * i] = A[g * 16 + t + 4 * i];
      a[2 * i + 1] = A[(g + 8) * 16 + t + 4 * i];
      b[i] = B[(t + 4 * i) * 8 + g];
    }
    m16n8k16(d, a, b);
  }
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

template <int SHAPE, int CHAINS>
__global__ void rate(int iters, unsigned long long* out, double* sink) {
  double d[CHAINS][4];
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.0;
  const double v = 1.0 + threadIdx.x * 1e-9;
  double a8[8] = {v, v, v, v, v, v, v, v}, b4[4] = {v, v, v, v};
  double a4[4] = {v, v, v, v}, b2[2] = {v, v}, a2[2] = {v, v};
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (SHAPE == 0) {
        double dd[2] = {d[c][0], d[c][1]};
        m8n8k4(dd, v, v);
        d[c][0] = dd[0]; d[c][1] = dd[1];
      } else if (SHAPE == 1) m16n8k4(d[c], a2, v);
      else if (SHAPE == 2) m16n8k8(d[c], a4, b2);
      else m16n8k16(d[c], a8, b4);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][3];
  if (s == 12345.678) sink[0] = s;
}

int main() {
  std::vector<double> A(256), B(128);
  for (int i = 0; i < 256; ++i) A[i] = (i * 37 % 101) * 0.25 - 3;
  for (int i = 0; i < 128; ++i) B[i] = (i * 53 % 97) * 0.5 - 7;
  double *dA, *dB, *dD;
  cudaMalloc(&dA, 256 * 8); cudaMalloc(&dB, 128 * 8); cudaMalloc(&dD, 128 * 8);
  cudaMemcpy(dA, A.data(), 256 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 128 * 8, cudaMemcpyHostToDevice);
  const char* names[] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const int Ks[] = {4, 4, 8, 16};
  for (int shape = 1; shape <= 3; ++shape) {
    layout_check<<<1, 32>>>(dA, dB, dD, shape);
    std::vector<double> D(128);
    cudaMemcpy(D.data(), dD, 128 * 8, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < 16; ++m)
      for (int n = 0; n < 8; ++n) {
        double r = 0;
        for (int k = 0; k < Ks[shape]; ++k) r += A[m * 16 + k] * B[k * 8 + n];
        err = fmax(err, fabs(r - D[m * 8 + n]));
      }
    printf("layout %s: max err %g (%s)\n", names[shape], err, cudaGetErrorString(cudaGetLastError()));
  }
  unsigned long long* out;
  double* sink;
  cudaMalloc(&out, 148 * 8 * 4); cudaMalloc(&sink, 8);
  const int iters = 4096;
  auto run = [&](auto kern, int shape, int warps, int chains) {
    kern<<<148, warps * 32>>>(iters, out, sink);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / (iters * chains * warps);  // cycles per instr per SM
    const double flops = 2.0 * (shape == 0 ? 8 * 8 * 4 : 16 * 8 * Ks[shape]);
    printf("%-9s warps %2d chains %d: %.2f cyc/instr/SM -> %.1f TFLOP/s @1.965GHz x148 (%s)\n", names[shape],
           warps, chains, per, flops / per * 1.965e9 * 148 / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  for (int w : {4, 8, 16}) {
    run(rate<0, 4>, 0, w, 4);
    run(rate<1, 4>, 1, w, 4);
    run(rate<2, 4>, 2, w, 4);
    run(rate<3, 4>, 3, w, 4);
  }
  return 0;
}
