// Microbenchmark: back-to-back tcgen05.mma throughput (kind::tf32 and kind::f16)
// with SWIZZLE_128B K-major operands resident in smem.  One CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1710_08124_b200/csrc tools/mma_bench.cu -o /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include <string>
#include "tc.cuh"

using namespace fepll;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc) : "memory");
}

// whole warp executes; one elected lane issues
__device__ __forceinline__ void mma_tf32_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "elect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ void mma_i8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "elect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc) : "memory");
}

// kind::i8: S32 accumulate (c_format 2), signed A and B (formats 1), K-major, K = 32
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void bench(int kind, int N, int iters, unsigned long long* out, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)base)[i] = 0.001f * (i % 7);
  if (threadIdx.x < 32) tc::tmem_alloc(&tmem, 512);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (kind == 3 && threadIdx.x < 32) {
    const uint32_t A = tc::smem_u32(base), B = tc::smem_u32(base + 32768);
    const uint32_t idi = idesc_i8(128, N);
    const uint64_t da = tc::desc_sw128(A), db = tc::desc_sw128(B);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tmem + ((kk % nacc) * 128);
        mma_i8_elect(d, da + 2 * kk, db + 2 * kk, idi, it | kk);
      }
    }
    if (threadIdx.x == 0) { tc::mma_commit(&bar); tc::mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if ((kind == 4 || kind == 5) && threadIdx.x < 32) {
    // A operand from tensor memory (TS form): kind 4 tf32 (K = 8: 8 columns), kind 5 bf16 (K = 16: 8 columns)
    const uint32_t B = tc::smem_u32(base + 32768);
    const uint32_t id = kind == 4 ? tc::idesc_tf32(128, N) : tc::idesc_bf16(128, N);
    const uint64_t db = tc::desc_sw128(B);
    const uint32_t a0 = tmem + 384;  // A columns beside the accumulators (uninitialised: timing only)
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tmem + ((kk % nacc) * 128);
        if (kind == 4) tc::mma_tf32_tmemA_warp(d, a0 + 8 * kk, db + 2 * kk, id, it | kk);
        else tc::mma_bf16_tmemA_warp(d, a0 + 8 * kk, db + 2 * kk, id, it | kk);
      }
    }
    if (threadIdx.x == 0) { tc::mma_commit(&bar); tc::mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (kind >= 10 && kind <= 15 && threadIdx.x < 32) {
    // whole-tile issue patterns (cycles per TILE reported as cycles/MMA x 1):
    //  10 ws2 tile: 8 SS tf32 N then 8 TS bf16 N, accumulators rotating over 3
    //  11 ws2 tile, SS / TS alternating
    //  12 Wiener tile (2 sets): 8 SS tf32 N=64, 8 TS tf32 N=32 (acc A); 4 TS tf32 N=128, 4 TS tf32 N=64 (acc B)
    //  13 Wiener tile, first product SS / TS alternating
    //  14 Wiener tile, second product's 8 TS interleaved with the NEXT tile's 8 SS (then that tile's 8 TS)
    //  15 Wiener tile with every TS replaced by SS of the same shape (what an smem A operand would cost)
    const uint32_t A = tc::smem_u32(base), B = tc::smem_u32(base + 32768);
    const uint64_t da = tc::desc_sw128(A), db = tc::desc_sw128(B);
    const uint32_t a0 = tmem + 448;
    const uint32_t idb = tc::idesc_bf16(128, N), idt = tc::idesc_tf32(128, N);
    const uint32_t i64 = tc::idesc_tf32(128, 64), i32 = tc::idesc_tf32(128, 32), i128 = tc::idesc_tf32(128, 128);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (it % 3) * 128;
      const uint32_t dA = tmem + (it & 1) * 192, dB = dA + 64;
      if (kind == 10) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc::mma_tf32_warp(d, da + 2 * (kk & 3), db + 2 * (kk & 3), idt, kk);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc::mma_bf16_tmemA_warp(d, a0 + 8 * kk, db + 2 * (kk & 3), idb, 1u);
      } else if (kind == 11) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          tc::mma_tf32_warp(d, da + 2 * (kk & 3), db + 2 * (kk & 3), idt, kk);
          tc::mma_bf16_tmemA_warp(d, a0 + 8 * kk, db + 2 * (kk & 3), idb, 1u);
        }
      } else if (kind == 12 || kind == 15) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc::mma_tf32_warp(dA, da + 2 * (kk & 3), db + 2 * (kk & 3), i64, kk);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (kind == 12) tc::mma_tf32_tmemA_warp(dA, a0 + 8 * kk, db + 2 * (kk & 3), i32, 1u);
          else tc::mma_tf32_warp(dA, da + 2 * (kk & 3), db + 2 * (kk & 3), i32, 1u);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (kind == 12) tc::mma_tf32_tmemA_warp(dB, a0 + 8 * kk, db + 2 * kk, i128, kk);
          else tc::mma_tf32_warp(dB, da + 2 * kk, db + 2 * kk, i128, kk);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (kind == 12) tc::mma_tf32_tmemA_warp(dB, a0 + 8 * kk, db + 2 * kk, i64, 1u);
          else tc::mma_tf32_warp(dB, da + 2 * kk, db + 2 * kk, i64, 1u);
        }
      } else if (kind == 13) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          tc::mma_tf32_warp(dA, da + 2 * (kk & 3), db + 2 * (kk & 3), i64, kk);
          tc::mma_tf32_tmemA_warp(dA, a0 + 8 * kk, db + 2 * (kk & 3), i32, 1u);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::mma_tf32_tmemA_warp(dB, a0 + 8 * kk, db + 2 * kk, i128, kk);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::mma_tf32_tmemA_warp(dB, a0 + 8 * kk, db + 2 * kk, i64, 1u);
      } else {  // 14
        const uint32_t dAn = tmem + ((it + 1) & 1) * 192;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          tc::mma_tf32_tmemA_warp(dB, a0 + 8 * (kk & 3), db + 2 * (kk & 3), kk < 4 ? i128 : i64, kk);
          tc::mma_tf32_warp(dAn, da + 2 * (kk & 3), db + 2 * (kk & 3), i64, kk);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc::mma_tf32_tmemA_warp(dAn, a0 + 8 * kk, db + 2 * (kk & 3), i32, 1u);
      }
    }
    if (threadIdx.x == 0) { tc::mma_commit(&bar); tc::mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if ((kind == 8 || kind == 9) && threadIdx.x < 32) {
    // alternating TS bf16 and SS tf32 on the SAME accumulator (one tile's main + cross passes interleaved);
    // kind 9: all SS first, then all TS (the ws2 order), same accumulator
    const uint32_t A = tc::smem_u32(base), B = tc::smem_u32(base + 32768);
    const uint32_t idb = tc::idesc_bf16(128, N), idt = tc::idesc_tf32(128, N);
    const uint64_t da = tc::desc_sw128(A), db = tc::desc_sw128(B);
    const uint32_t a0 = tmem + 384;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (it % nacc) * 128;
      if (kind == 8) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          tc::mma_tf32_warp(d, da + 2 * kk, db + 2 * kk, idt, kk);
          tc::mma_bf16_tmemA_warp(d, a0 + 8 * kk, db + 2 * kk, idb, 1u);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::mma_tf32_warp(d, da + 2 * kk, db + 2 * kk, idt, kk);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc::mma_bf16_tmemA_warp(d, a0 + 8 * kk, db + 2 * kk, idb, 1u);
      }
    }
    if (threadIdx.x == 0) { tc::mma_commit(&bar); tc::mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if ((kind == 6 || kind == 7) && threadIdx.x < 32) {
    // alternating TS bf16 (accumulator 0) and SS tf32 (accumulator 1): do the SS MMAs hide in the TS latency?
    // kind 7: two SS per TS
    const uint32_t A = tc::smem_u32(base), B = tc::smem_u32(base + 32768);
    const uint32_t idb = tc::idesc_bf16(128, N), idt = tc::idesc_tf32(128, N);
    const uint64_t da = tc::desc_sw128(A), db = tc::desc_sw128(B);
    const uint32_t a0 = tmem + 384;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        tc::mma_bf16_tmemA_warp(tmem, a0 + 8 * kk, db + 2 * kk, idb, it | kk);
        tc::mma_tf32_warp(tmem + 128, da + 2 * kk, db + 2 * kk, idt, it | kk);
        if (kind == 7) tc::mma_tf32_warp(tmem + 256, da + 2 * kk, db + 2 * kk, idt, it | kk);
      }
    }
    if (threadIdx.x == 0) { tc::mma_commit(&bar); tc::mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (kind == 2 && threadIdx.x < 32) {
    const uint32_t A = tc::smem_u32(base), B = tc::smem_u32(base + 32768);
    const uint32_t idt = tc::idesc_tf32(128, N);
    const uint64_t da = tc::desc_sw128(A), db = tc::desc_sw128(B);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tmem + ((kk % nacc) * 128);
        mma_tf32_elect(d, da + 2 * kk, db + 2 * kk, idt, it | kk);
      }
    }
    if (threadIdx.x == 0) { tc::mma_commit(&bar); tc::mbar_wait(&bar, 0); }
    __syncwarp();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (kind < 2 && threadIdx.x == 0) {
    const uint32_t A = tc::smem_u32(base), B = tc::smem_u32(base + 32768);
    const uint32_t idt = tc::idesc_tf32(128, N);
    // f16: c_format F32 (1<<4), a/b format F16 (0), K-major
    const uint32_t idh = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tmem + ((it * 4 + kk) % nacc) * 128;
        if (kind == 0)
          tc::mma_tf32(d, tc::desc_sw128(A + kk * 32), tc::desc_sw128(B + kk * 32), idt, it | kk);
        else
          mma_f16(d, tc::desc_sw128(A + kk * 32), tc::desc_sw128(B + kk * 32), idh, it | kk);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (argc > 1 && std::string(argv[1]) == "--peak") {
    // dense TF32 / BF16 peak on all 148 SMs, CUDA-event timed: a short burst
    // and a ~2 s sustained run (power-capped clocks), M128 x N256 MMAs
    for (int kind : {2, 1, 3}) {
      for (int iters : {4000, 400000}) {
        bench<<<148, 128, 80 * 1024>>>(kind, 256, 100, d, 1);  // warm-up
        cudaEventRecord(e0);
        bench<<<148, 128, 80 * 1024>>>(kind, 256, iters, d, 1);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 148.0 * iters * 4 * 2.0 * 128 * 256 * (kind == 1 ? 16 : kind == 3 ? 32 : 8);
        printf("{\"kind\": \"%s\", \"iters\": %d, \"ms\": %.3f, \"tflops\": %.1f, \"status\": \"%s\"}\n",
               kind == 1 ? "f16" : kind == 3 ? "i8" : "tf32", iters, ms, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
      }
    }
    return 0;
  }
  for (int nacc : {1, 2, 4})
  for (int kind = 0; kind < 16; ++kind)
    for (int N : {32, 64, 128, 256}) {
      if (N == 256 && nacc > 2) continue;
      if ((kind == 6 || kind == 7) && (N > 128 || nacc > 1)) continue;
      if ((kind == 8 || kind == 9) && (N > 128 || nacc > 3)) continue;
      if (kind >= 10 && (nacc > 1 || ((kind == 10 || kind == 11) ? (N != 128 && N != 64) : N != 32))) continue;
      const int iters = 2000;
      bench<<<148, 128, 80 * 1024>>>(kind, N, iters, d, N == 256 ? 1 : nacc);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = (double)h[0] / (iters * (kind >= 10 ? 1 : 4));
      double macs = 128.0 * N * ((kind == 1 || kind == 5) ? 16 : kind == 3 ? 32 : 8);
      printf("nacc=%d %s N=%3d: %.1f cycles/MMA  -> %.0f MAC/clk/SM (%s)\n", nacc, kind == 0 ? "tf32" : (kind == 1 ? "f16 " : kind == 3 ? "i8  " : kind == 4 ? "tf32E-TS" : kind == 5 ? "bf16E-TS" : kind == 6 ? "TS+SS pair" : kind == 7 ? "TS+2SS trio" : kind == 8 ? "SS,TS alternating same acc (per pair)" : kind == 9 ? "4 SS then 4 TS same acc (per pair)" : kind == 10 ? "ws2 tile 8SS+8TS (cycles per tile)" : kind == 11 ? "ws2 tile alternating (per tile)" : kind == 12 ? "wiener tile 8SS+8TS | 8TS (per tile)" : kind == 13 ? "wiener tile G1 alternating (per tile)" : kind == 14 ? "wiener tile G2(i) x G1ss(i+1) interleaved (per tile)" : kind == 15 ? "wiener tile all SS (per tile)" : "tf32E"),
             N, cyc, macs / cyc, cudaGetErrorString(e));
    }
  return 0;
}
