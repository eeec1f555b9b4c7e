// Do FP64 mma.sync (DMMA) and scalar DFMA share one pipe on sm_100a?
// Warps [0, wd) run m8n8k4 DMMA chains, warps [wd, w) run DFMA chains; the
// combined FP64 rate tells whether a Wiener kernel could add DFMA work next
// to its DMMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/fp64_mix_bench.cu -o tools/fp64_mix_bench
#include <cstdio>

__device__ __forceinline__ void m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int kChains = 8;

__global__ void mix(int iters, int wd, unsigned long long* cyc, double* sink, unsigned long long* wt) {
  const int warp = threadIdx.x >> 5;
  double d[kChains][2];
  const double v = 1.0 + threadIdx.x * 1e-9, u = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = c * 1e-3;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < wd) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) m8n8k4(d[c][0], d[c][1], v, u);
    }
  } else {
    // per thread 2 DFMA per chain step = 4 flops; a DMMA step is 512 flops per warp = 16 per thread
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        d[c][0] = fma(d[c][0], v, u);
        d[c][1] = fma(d[c][1], u, v);
      }
    }
  }
  const unsigned long long tw = clock64();
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) wt[warp] = tw - t0;
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) sink[0] = s;
}

int main() {
  unsigned long long* cyc;
  double* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 8);
  unsigned long long* wt;
  cudaMalloc(&wt, 32 * 8);
  const int iters = 2048;
  auto run = [&](int w, int wd) {
    mix<<<148, w * 32>>>(iters, wd, cyc, sink, wt);
    cudaDeviceSynchronize();
    unsigned long long h, hw[32];
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hw, wt, w * 8, cudaMemcpyDeviceToHost);
    unsigned long long md = 0, mf = 0;
    for (int i = 0; i < w; ++i) (i < wd ? md : mf) = hw[i] > (i < wd ? md : mf) ? hw[i] : (i < wd ? md : mf);
    printf("   per-warp max cycles: dmma %llu dfma %llu\n", md, mf);
    // every warp does the same flop count: iters * kChains * 512
    const double flops_sm = (double)w * iters * kChains * 512.0;
    printf("warps %2d (dmma %2d, dfma %2d): %8llu cycles  %.1f flop/cycle/SM -> %.1f TFLOP/s @1.9GHz x148 (%s)\n",
           w, wd, w - wd, h, flops_sm / h, flops_sm / h * 1.9e9 * 148 / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int w : {4, 8, 12}) run(w, 0);
  for (int w : {8, 16}) {
    run(w, w);
    run(w, 0);
    run(w, w / 2);
  }
  run(16, 12);
  run(16, 4);
  return 0;
}
