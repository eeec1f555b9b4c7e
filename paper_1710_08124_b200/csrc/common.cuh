// Shared helpers for the FEPLL sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

namespace fepll {

constexpr int kOk = 0;
constexpr int kDataError = 3;
constexpr int kNumericalError = 4;
constexpr int kDeviceError = 5;

constexpr int kMaxP = 256;          // side <= 16
constexpr int kMaxGroupCols = 512;  // sum of child ranks of one node (TMEM width)
constexpr int kMaxChildren = 32;
constexpr int kMaxDepth = 64;
constexpr int kSMs = 148;

void set_error(const std::string& msg);
void count_launch();

#define FEPLL_CUDA(expr)                                                        \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::fepll::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));   \
      return ::fepll::kDeviceError;                                             \
    }                                                                           \
  } while (0)

#define FEPLL_LAUNCH()                                                          \
  do {                                                                          \
    ::fepll::count_launch();                                                    \
    cudaError_t _e = cudaGetLastError();                                        \
    if (_e != cudaSuccess) {                                                    \
      ::fepll::set_error(std::string("launch: ") + cudaGetErrorString(_e));     \
      return ::fepll::kDeviceError;                                             \
    }                                                                           \
  } while (0)

#define FEPLL_REQUIRE(cond, msg)                                                \
  do {                                                                          \
    if (!(cond)) {                                                              \
      ::fepll::set_error(msg);                                                  \
      return ::fepll::kDataError;                                               \
    }                                                                           \
  } while (0)

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int grid_for(int64_t items, int per_block, int cap = 148 * 16) {
  int64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

}  // namespace fepll
