// Shared helpers for the FEPLL sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

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
constexpr int kLeafSlack = 32;  // extra leaf-bucket slots per leaf (deferred verification re-routes)

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

// Programmatic dependent launch (PDL): a kernel launched with
// launch_pdl may start (prologue: TMEM, barriers) while its stream
// predecessor drains; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible — call it before touching any data the
// predecessor produces or reads.  pdl_trigger() lets this grid's own
// dependents begin launching.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline int grid_for(int64_t items, int per_block, int cap = 148 * 16) {
  int64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

}  // namespace fepll
