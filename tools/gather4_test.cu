// Check TMA tile::gather4 with SWIZZLE_128B lands rows in the canonical
// K-major swizzled layout (chunk c of row r at (c ^ (r % 8)) * 16).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1710_08124_b200/csrc tools/gather4_test.cu -o /tmp/g4 -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "tc.cuh"

using namespace fepll;

__global__ void k(const __grid_constant__ CUtensorMap map, const int* rows, float* out) {
  __shared__ __align__(1024) float sm[8 * 32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::mbar_arrive_expect_tx(&bar, 8 * 128);
    for (int h = 0; h < 2; ++h) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(tc::smem_u32(sm + h * 128)),
          "l"(&map), "r"(0), "r"(rows[4 * h]), "r"(rows[4 * h + 1]), "r"(rows[4 * h + 2]),
          "r"(rows[4 * h + 3]), "r"(tc::smem_u32(&bar))
          : "memory");
    }
  }
  tc::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int R = 64, C = 64;
  std::vector<float> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = r * 1000 + c;
  float* d;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)rc);
  int hr[8] = {5, 17, 2, 63, 40, 41, 0, 9};
  int* dr;
  cudaMalloc(&dr, 32);
  cudaMemcpy(dr, hr, 32, cudaMemcpyHostToDevice);
  float* dout;
  cudaMalloc(&dout, 256 * 4);
  k<<<1, 128>>>(map, dr, dout);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> o(256);
  cudaMemcpy(o.data(), dout, 1024, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 32; ++c) {
      const int chunk = c / 4, within = c % 4;
      const float got = o[r * 32 + ((chunk ^ (r % 8)) * 4) + within];
      const float want = hr[r] * 1000 + c;
      if (got != want) ++bad;
    }
  printf("swizzled-layout mismatches: %d / 256\n", bad);
  return 0;
}
