// Microbenchmark: issue cost of staging 128-row tiles of random 256-byte
// FP32 rows (the select_ws2.cu producer's job) with no consumer attached.
//   0  cp.async 16 B (LDGSTS.128), 8 warps, lanes 8r..8r+7 = one row's atom,
//      four stages, wait_group<2> per tile (the ws2 producer loop)
//   1  same, 16 warps (half the instructions per warp)
//   2  1-D bulk copy (cp.async.bulk) of the whole 256-byte row, rows split
//      over the 32 lanes of one warp, mbarrier completion
//   3  same, issued by lane 0 only
//   4  variant 0 with 4 warps, 5: with 2 warps
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1710_08124_b200/csrc tools/ldgsts_rate.cu -o /tmp/ldgsts_rate
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "tc.cuh"

using namespace fepll;

constexpr int kRows = 128;
constexpr int kRowBytes = 256;
constexpr int kTileBytes = kRows * kRowBytes;
constexpr int kStages = 4;

template <int V>
__global__ void __launch_bounds__(512, 1)
bench(const float* data, const int* rows, int ntile, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = tc::align1024(sm);
  __shared__ uint64_t full[kStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) tc::mbar_init(&full[i], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int* my = rows + (size_t)blockIdx.x * ntile * kRows;
  const unsigned long long t0 = clock64();
  if (V == 0 || V == 1 || V >= 4) {
    constexpr int kWarps = V == 0 ? 8 : V == 1 ? 16 : V == 4 ? 4 : 2;
    if (warp < kWarps) {
      // warp w: atom w % 2, rows (w / 2) * (256 / kWarps) ..
      const int ka = warp & 1;
      const int rpw = 2 * kRows / kWarps;          // rows per warp
      const int r0 = (warp >> 1) * rpw;
      auto issue = [&](int i) {
        if (i >= ntile) return;
        uint8_t* stg = base + (i % kStages) * kTileBytes + ka * (kRows * 128);
        const int* ri = my + (size_t)i * kRows + r0;
        int g[32];
#pragma unroll
        for (int q = 0; q < rpw / 4; ++q) g[q] = ri[4 * q + (lane >> 3)];
#pragma unroll
        for (int q = 0; q < rpw / 4; ++q) {
          const int r = r0 + 4 * q + (lane >> 3);
          const int c = lane & 7;
          tc::cp_async16(stg + (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4),
                         data + (int64_t)g[q] * 64 + ka * 32 + 4 * c);
        }
      };
      for (int j = 0; j < kStages - 1; ++j) { issue(j); tc::cp_async_commit(); }
      for (int i = 0; i < ntile; ++i) {
        tc::cp_async_wait<kStages - 2>();
        __syncwarp();
        issue(i + kStages - 1);
        tc::cp_async_commit();
      }
      tc::cp_async_wait<0>();
    }
  } else if (warp == 0) {
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      if (i >= kStages) tc::mbar_wait(&full[st], ((i / kStages) - 1) & 1);
      uint8_t* A = base + st * kTileBytes;
      const int* ri = my + (size_t)i * kRows;
      if (lane == 0) tc::mbar_arrive_expect_tx(&full[st], kTileBytes);
      __syncwarp();
      if (V == 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = 32 * q + lane;
          tc::bulk_g2s(A + r * kRowBytes, data + (int64_t)ri[r] * 64, kRowBytes, &full[st]);
        }
      } else if (lane == 0) {
        for (int r = 0; r < kRows; ++r)
          tc::bulk_g2s(A + r * kRowBytes, data + (int64_t)ri[r] * 64, kRowBytes, &full[st]);
      }
      __syncwarp();
    }
    for (int st = 0; st < kStages; ++st) {
      const int last = ntile - kStages + st;
      if (last >= 0) tc::mbar_wait(&full[last % kStages], (last / kStages) & 1);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  const size_t R = (size_t)1 << 22;  // 4M rows x 256 B = 1 GiB
  float* d;
  cudaMalloc(&d, R * kRowBytes);
  cudaMemset(d, 0, R * kRowBytes);
  const int ntile = 220;  // one tree level of cfg5 per SM
  std::vector<int> h((size_t)148 * ntile * kRows);
  int* dr;
  cudaMalloc(&dr, h.size() * 4);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  const int smem = kStages * kTileBytes + 1024;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      kern<<<148, 512, smem>>>(d, dr, ntile, out);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> o(148);
      cudaMemcpy(o.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%-26s: %5.0f ns/tile, %.2f TB/s (%s)\n", name, ms * 1e6 / ntile,
                      148.0 * ntile * kTileBytes / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    }
  };
  std::mt19937 g(1);
  for (int mode = 0; mode < 2; ++mode) {
    for (size_t k = 0; k < h.size(); ++k) h[k] = mode == 0 ? (int)(g() % R) : (int)(k % R);
    cudaMemcpy(dr, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    printf("%s rows\n", mode == 0 ? "random" : "sequential");
    run(bench<0>, "cp.async16 8 warps");
    run(bench<1>, "cp.async16 16 warps");
    run(bench<2>, "bulk 256B 32 lanes");
    run(bench<3>, "bulk 256B lane 0");
    run(bench<4>, "cp.async16 4 warps");
    run(bench<5>, "cp.async16 2 warps");
  }
  return 0;
}
