// Microbenchmark: how fast can one CTA per SM pull 128-row tiles of random
// 128-byte row atoms into shared memory?  Variants:
//   0 gather4, issued by all 32 lanes (compiler waterfall)
//   1 gather4, issued by lane 0, row indices read from smem
//   2 2-D tile box {32 floats, 4 rows} (contiguous rows, same bytes/instr)
//   3 2-D tile box {32 floats, 32 rows}
//   4 1-D bulk copy, 128 B per row, lane 0
//   5 LDG.128 -> STS by 256 threads (register staging, one tile ahead)
// Rows are random indices into a 1 GiB FP32 array (HBM-resident).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1710_08124_b200/csrc tools/tma_rate.cu -o /tmp/tma_rate
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "tc.cuh"

using namespace fepll;

constexpr int kRowsPerTile = 128;
constexpr int kAtoms = 4;                    // 4 x 128 B per row = 64 KB per tile
constexpr int kTileBytes = kRowsPerTile * kAtoms * 128;
constexpr int kStages = 2;

__device__ __forceinline__ void g4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                   int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(tc::smem_u32(dst)),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tile2d(void* dst, const CUtensorMap* map, int col, int row, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(tc::smem_u32(dst)),
      "l"(map), "r"(col), "r"(row), "r"(tc::smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(256, 1)
bench(int variant, const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m4,
      const __grid_constant__ CUtensorMap m32, const float* data, const int* rows, int ntile,
      unsigned long long* out, int pitch) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages];
  __shared__ int sidx[kStages][kRowsPerTile];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1); }
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int* my = rows + (size_t)blockIdx.x * ntile * kRowsPerTile;
  unsigned long long t0 = clock64();
  if (variant == 5) {
    // 256 threads: thread t loads row t/2, half (t&1) -> 2 atoms = 16 x 16 B
    const int r = tid >> 1, h = tid & 1;
    float4 v[16];
    auto load = [&](int i) {
      const float4* src = reinterpret_cast<const float4*>(data + (size_t)my[i * kRowsPerTile + r] * pitch) + h * 16;
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = __ldg(src + c);
    };
    load(0);
    for (int i = 0; i < ntile; ++i) {
      uint8_t* A = base + (i % kStages) * kTileBytes;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int atom = h * 2 + c / 8, ch = c % 8;
        *reinterpret_cast<float4*>(A + atom * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4)) = v[c];
      }
      __syncthreads();
      if (i + 1 < ntile) load(i + 1);
    }
  } else if (warp == 0) {
    for (int i = 0; i < ntile; ++i) {
      const int st = i % kStages;
      // no consumer: the stage is free once its previous fill landed
      if (i >= kStages) tc::mbar_wait(&full[st], ((i / kStages) - 1) & 1);
      uint8_t* A = base + st * kTileBytes;
      const int* ri = my + (size_t)i * kRowsPerTile;
      if (variant == 1 || variant == 4) {
        sidx[st][lane] = ri[lane]; sidx[st][lane + 32] = ri[lane + 32];
        sidx[st][lane + 64] = ri[lane + 64]; sidx[st][lane + 96] = ri[lane + 96];
        __syncwarp();
      }
      if (lane == 0) tc::mbar_arrive_expect_tx(&full[st], kTileBytes);
      __syncwarp();
      if (variant == 0) {
        const int r0 = ri[4 * lane], r1 = ri[4 * lane + 1], r2 = ri[4 * lane + 2], r3 = ri[4 * lane + 3];
        const int off = (lane >> 1) * 1024 + (lane & 1) * 512;
        for (int a = 0; a < kAtoms; ++a) g4(A + a * 16384 + off, &m1, a * 32, r0, r1, r2, r3, &full[st]);
      } else if (variant == 1 && lane == 0) {
        for (int j = 0; j < 32; ++j) {
          const int off = (j >> 1) * 1024 + (j & 1) * 512;
          const int r0 = sidx[st][4 * j], r1 = sidx[st][4 * j + 1], r2 = sidx[st][4 * j + 2], r3 = sidx[st][4 * j + 3];
          for (int a = 0; a < kAtoms; ++a) g4(A + a * 16384 + off, &m1, a * 32, r0, r1, r2, r3, &full[st]);
        }
      } else if (variant == 2 && lane == 0) {
        for (int j = 0; j < 32; ++j)
          for (int a = 0; a < kAtoms; ++a)
            tile2d(A + a * 16384 + j * 512, &m4, a * 32, (ri[0] + 4 * j) & ~3, &full[st]);
      } else if (variant == 3 && lane == 0) {
        for (int j = 0; j < 4; ++j)
          for (int a = 0; a < kAtoms; ++a)
            tile2d(A + a * 16384 + j * 4096, &m32, a * 32, (ri[0] + 32 * j) & ~31, &full[st]);
      } else if (variant == 4 && lane == 0) {
        for (int j = 0; j < 128; ++j)
          for (int a = 0; a < kAtoms; ++a)
            tc::bulk_g2s(A + a * 16384 + j * 128, data + (size_t)sidx[st][j] * pitch + a * 32, 128, &full[st]);
      }
      __syncwarp();
    }
    for (int st = 0; st < kStages; ++st) {
      const int last = ntile - kStages + st;  // last use of stage (last % kStages)
      if (last >= 0) tc::mbar_wait(&full[last % kStages], (last / kStages) & 1);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

// massively parallel random-row gather: 16 lanes per 256-byte row segment
__global__ void gather_ldg(const float* data, const int* rows, size_t nrows_total, int pitch, float4* out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t r = t >> 4;
  if (r >= nrows_total) return;
  const int c = t & 15;
  out[t] = __ldg(reinterpret_cast<const float4*>(data + (size_t)rows[r] * pitch) + c);
}

static void make_map(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, float* d, size_t R, int C, int boxr) {
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)boxr};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc) printf("encode failed %d\n", (int)rc);
}

int main() {
  const int C = 128;                         // floats per row (512 B, 4 atoms)
  const size_t R = (size_t)1 << 21;          // 2M rows x 512 B = 1 GiB
  float* d;
  cudaMalloc(&d, R * C * 4);
  cudaMemset(d, 0, R * C * 4);
  const int ntile = 400;
  std::vector<int> h((size_t)148 * ntile * kRowsPerTile);
  std::mt19937 g(1);
  for (auto& x : h) x = g() % R;
  int* dr;
  cudaMalloc(&dr, h.size() * 4);
  cudaMemcpy(dr, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m1, m4, m32;
  make_map(enc, &m1, d, R, C, 1);
  make_map(enc, &m4, d, R, C, 4);
  make_map(enc, &m32, d, R, C, 32);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  const int smem = kStages * kTileBytes + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"gather4 32-lane", "gather4 lane0", "tile box 4 rows", "tile box 32 rows", "bulk 128B lane0",
                         "LDG->STS 256 thr"};
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 6; ++v) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      bench<<<148, 256, smem>>>(v, m1, m4, m32, d, dr, ntile, out, C);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> o(148);
      cudaMemcpy(o.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
      double bytes = 148.0 * ntile * kTileBytes;
      printf("%-18s: %.0f cyc/tile (64 KB) CTA0, %.2f TB/s chip (%s)\n", names[v], (double)o[0] / ntile,
             bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    }
  // random 256 B rows (first half of each 512 B row), HBM vs L2-resident
  float4* o2;
  const size_t nr = (size_t)148 * ntile * kRowsPerTile;
  cudaMalloc(&o2, nr * 256);
  for (size_t span : {R, (size_t)1 << 16, (size_t)1 << 17}) {
    for (auto& x : h) x = g() % span;
    cudaMemcpy(dr, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      gather_ldg<<<(unsigned)((nr * 16 + 255) / 256), 256>>>(d, dr, nr, C, o2);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("LDG gather 256B rows, span %zu rows (%zu MB): read %.2f TB/s (+write same) (%s)\n", span,
             span * 512 >> 20, nr * 256 / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    }
  }
  return 0;
}
