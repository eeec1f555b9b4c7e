// Offline search-tree construction on the device:
// the two O(K^2 P^2) / O(sweeps K^2) parts of the reference's build_tree.
//
//  * fepll_tree_kl — pairwise symmetric KL of K flat-tail components
//    (pkg/src/fepll/tree.py:99-107): t[a][b] = Tr(C_a^-1 C_b) as a K x K
//    matrix product of the flattened inverses and covariances (C_b is
//    symmetric, so Tr(C_a^-1 C_b) = <C_a^-1, C_b> over P^2 entries), then
//    kl = 0.5 (t + t^T) - P with a zero diagonal, in the reference's
//    operation order.  FP64 throughout; one CTA per (a, 16-wide b tile).
//  * fepll_cluster_swap — the pairwise-swap local search of
//    balanced_cluster (pkg/src/fepll/tree.py:176-198), exactly sequential:
//    for each i the CTA evaluates every candidate j > i at once under the
//    current assignment, takes the FIRST improving j (the reference's scan
//    order), applies that swap (cluster ids + the two touched rowsum
//    columns, one thread per row) and resumes the scan at j + 1.  The delta
//    and rowsum updates use the reference's left-to-right FP64 operations
//    without contraction, so the result is the reference's partition.
#include <cstdint>

#include "common.cuh"

namespace fepll {

namespace tb {
constexpr int kThreads = 256;
constexpr int kBTile = 16;

// t[a][b] = sum_e inv[a][e] * cov[b][e], e over P^2; 16 b per CTA
__global__ void __launch_bounds__(kThreads)
trace_product_kernel(const double* __restrict__ inv, const double* __restrict__ cov, int K, int64_t P2,
                     double* __restrict__ t) {
  const int a = blockIdx.x;
  const int b0 = blockIdx.y * kBTile;
  const double* ia = inv + (int64_t)a * P2;
  double acc[kBTile];
#pragma unroll
  for (int q = 0; q < kBTile; ++q) acc[q] = 0.0;
  for (int64_t e = threadIdx.x; e < P2; e += kThreads) {
    const double v = ia[e];
#pragma unroll
    for (int q = 0; q < kBTile; ++q)
      if (b0 + q < K) acc[q] = fma(v, cov[(int64_t)(b0 + q) * P2 + e], acc[q]);
  }
  __shared__ double red[kThreads / 32][kBTile];
#pragma unroll
  for (int q = 0; q < kBTile; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane_id() == 0) red[warp_id()][q] = s;
  }
  __syncthreads();
  if (threadIdx.x < kBTile && b0 + threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w][threadIdx.x];
    t[(int64_t)a * K + b0 + threadIdx.x] = s;
  }
}

// kl = 0.5 * (t + t^T) - P, diagonal 0 (tree.py:104-106)
__global__ void symmetrize_kernel(const double* __restrict__ t, int K, double P, double* __restrict__ kl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)K * K) return;
  const int a = (int)(idx / K), b = (int)(idx - (int64_t)a * K);
  const double s = __dadd_rn(t[(int64_t)a * K + b], t[(int64_t)b * K + a]);
  kl[idx] = a == b ? 0.0 : __dsub_rn(__dmul_rn(0.5, s), P);
}

// the swap delta of tree.py:183-185, left to right, no contraction
__device__ __forceinline__ double swap_delta(const double* rowsum, int L, const double* D, int n, int i,
                                             int j, int a, int b) {
  double d = __dsub_rn(rowsum[(int64_t)i * L + b], rowsum[(int64_t)i * L + a]);
  d = __dadd_rn(d, rowsum[(int64_t)j * L + a]);
  d = __dsub_rn(d, rowsum[(int64_t)j * L + b]);
  d = __dsub_rn(d, __dmul_rn(2.0, D[(int64_t)i * n + j]));
  return __dmul_rn(2.0, d);
}

__global__ void __launch_bounds__(kThreads)
cluster_swap_kernel(const double* __restrict__ D, int n, int L, int64_t* __restrict__ cid,
                    double* __restrict__ rowsum, int sweeps, int32_t* __restrict__ sweeps_done) {
  __shared__ int first[kThreads / 32];
  __shared__ int jpick;
  __shared__ int any_improved;
  int done = 0;
  for (int sw = 0; sw < sweeps; ++sw) {
    if (threadIdx.x == 0) any_improved = 0;
    __syncthreads();
    for (int i = 0; i < n; ++i) {
      int j0 = i + 1;
      while (j0 < n) {
        const int ci = (int)cid[i];
        int mine = n;
        for (int j = j0 + threadIdx.x; j < n; j += kThreads) {
          const int cj = (int)cid[j];
          if (cj != ci && swap_delta(rowsum, L, D, n, i, j, ci, cj) < -1e-12) {
            mine = j;
            break;  // later j of this thread are larger
          }
        }
        // block-wide minimum j
        for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(0xffffffffu, mine, o));
        if (lane_id() == 0) first[warp_id()] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
          int m = n;
          for (int w = 0; w < kThreads / 32; ++w) m = min(m, first[w]);
          jpick = m;
        }
        __syncthreads();
        const int j = jpick;
        if (j >= n) break;
        const int a = ci, b = (int)cid[j];
        // rowsum[:, a] += D[:, j] - D[:, i]; rowsum[:, b] += D[:, i] - D[:, j]
        for (int r = threadIdx.x; r < n; r += kThreads) {
          const double dj = D[(int64_t)r * n + j], di = D[(int64_t)r * n + i];
          rowsum[(int64_t)r * L + a] = __dadd_rn(rowsum[(int64_t)r * L + a], __dsub_rn(dj, di));
          rowsum[(int64_t)r * L + b] = __dadd_rn(rowsum[(int64_t)r * L + b], __dsub_rn(di, dj));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          cid[i] = b;
          cid[j] = a;
          any_improved = 1;
        }
        __syncthreads();
        j0 = j + 1;
      }
    }
    __syncthreads();
    ++done;
    if (!any_improved) break;
    __syncthreads();
  }
  if (threadIdx.x == 0 && sweeps_done) *sweeps_done = done;
}
}  // namespace tb

}  // namespace fepll

using namespace fepll;

extern "C" int fepll_tree_kl(const double* inv, const double* cov, int32_t K, int32_t P, double* t_scratch,
                             double* kl, void* stream) {
  FEPLL_REQUIRE(inv && cov && t_scratch && kl && K >= 1 && P >= 1, "tree_kl: bad arguments");
  FEPLL_REQUIRE(K <= 65535 * tb::kBTile, "tree_kl: too many components");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t P2 = (int64_t)P * P;
  dim3 grid(K, (K + tb::kBTile - 1) / tb::kBTile);
  tb::trace_product_kernel<<<grid, tb::kThreads, 0, st>>>(inv, cov, K, P2, t_scratch);
  FEPLL_LAUNCH();
  const int64_t KK = (int64_t)K * K;
  tb::symmetrize_kernel<<<(unsigned)((KK + 255) / 256), 256, 0, st>>>(t_scratch, K, (double)P, kl);
  FEPLL_LAUNCH();
  return kOk;
}

extern "C" int fepll_cluster_swap(const double* D, int32_t n, int32_t L, int64_t* cid, double* rowsum,
                                  int32_t sweeps, int32_t* sweeps_done, void* stream) {
  FEPLL_REQUIRE(D && cid && rowsum && n >= 1 && L >= 1 && sweeps >= 0, "cluster_swap: bad arguments");
  tb::cluster_swap_kernel<<<1, tb::kThreads, 0, (cudaStream_t)stream>>>(D, n, L, cid, rowsum, sweeps,
                                                                       sweeps_done);
  FEPLL_LAUNCH();
  return kOk;
}
