// Kernel (c): Wiener estimates on the FP64 tensor cores (DMMA).
//
// Restates pkg/src/fepll/gmm.py:352-359 for every patch of a leaf bucket
// (the grouping of pkg/src/fepll/solver.py:233-241):
//     C    = (Z U_k) * (gamma - gamma_tail)        64 x r
//     Zhat = C U_k^T + gamma_tail Z                64 x P
// in FP64 — the estimates become the next iteration's image, whose tree
// decisions must stay the FP64 reference's, so no reduced precision here.
//
// A CTA (8 warps) walks a contiguous range of 64-patch tiles in leaf order:
// U_k is staged in smem once per leaf, the FP64 patch rows (kernel (a)
// output, 512 B each) arrive by cp.async into a double buffer while the
// previous tile computes.  Both products run as mma.sync m8n8k4 f64:
// warp w owns rows 8w..8w+7 of the tile.
#include "route.cuh"

namespace fepll {

namespace wn {

constexpr int kRows = 64;
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxP = 128;
constexpr int kMaxR = 64;

struct Head {
  int32_t tpre[kMaxLevelNodes + 1];
  uint64_t scan_tmp[256];
  int32_t rows[2][kRows];
  int32_t t_begin, t_end;
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Row strides (in doubles) are chosen so every fragment load is two
// conflict-free shared-memory wavefronts: A-side tiles (rows g, 4
// consecutive k) use ld = 4 mod 16, B-side tiles (4 rows k, 8 consecutive n)
// use ld = 8 mod 16.
struct Geo {
  int P, Pn;     // P, P rounded up to 8 (phase-2 N)
  int zld;       // Zs [64][zld]
  int R8;        // rank rounded up to 8
  int uld;       // Us [Pn][uld]  (phase-1 B: k = p, n = j)
  int utld;      // UT [R8][utld] (phase-2 B: k = j, n = p)
  int cld;       // Cs [64][cld]
};

template <int NT2>  // phase-2 n-tiles (P/8 rounded up): 8 for P=64, 13 for P=100
__global__ void __launch_bounds__(kThreads)
wiener_dmma_kernel(PlanView pv, int t, const int32_t* __restrict__ leaf_nodes, int n_leaf_nodes,
                   const int32_t* __restrict__ cnt, const int64_t* __restrict__ off,
                   const int32_t* __restrict__ leafseg, const double* __restrict__ Z64,
                   double* __restrict__ Zhat, Geo geo) {
  extern __shared__ __align__(16) uint8_t smem[];
  Head& h = *reinterpret_cast<Head*>(smem);
  double* Zs0 = reinterpret_cast<double*>(smem + ((sizeof(Head) + 127) & ~size_t(127)));
  double* Zs1 = Zs0 + kRows * geo.zld;
  double* Us = Zs1 + kRows * geo.zld;          // [Pn][uld]   (p, j)
  double* UT = Us + geo.Pn * geo.uld;          // [R8][utld]  (j, p)
  double* Cs = UT + geo.R8 * geo.utld;         // [64][cld]
  double* sh = Cs + kRows * geo.cld;           // [R8]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = geo.P;
  for (int k = tid; k < n_leaf_nodes; k += kThreads)
    h.tpre[k] = (cnt[leaf_nodes[k]] + kRows - 1) / kRows;
  __syncthreads();
  const int tiles = block_exscan(h.tpre, n_leaf_nodes, h.scan_tmp);
  if (tid == 0) {
    h.tpre[n_leaf_nodes] = tiles;
    h.t_begin = (int)(((int64_t)tiles * blockIdx.x) / gridDim.x);
    h.t_end = (int)(((int64_t)tiles * (blockIdx.x + 1)) / gridDim.x);
  }
  __syncthreads();
  const int t_begin = h.t_begin, t_end = h.t_end;
  if (t_begin >= t_end) return;

  // stage the rows of tile `tile` into buffer b (cp.async, 16-byte chunks)
  auto issue_tile = [&](int tile, int b) {
    const int li = prefix_find(h.tpre, n_leaf_nodes, tile);
    const int v = leaf_nodes[li];
    const int first = (tile - h.tpre[li]) * kRows;
    const int m = min(kRows, cnt[v] - first);
    if (tid < kRows) h.rows[b][tid] = tid < m ? leafseg[off[v] + first + tid] : -1;
    __syncthreads();
    double* Zs = b ? Zs1 : Zs0;
    const int chunks = P / 2;  // 16-byte chunks per row (P even)
    for (int e = tid; e < kRows * chunks; e += kThreads) {
      const int i = e / chunks, c = e - i * chunks;
      const int g = h.rows[b][i];
      double* dst = Zs + i * geo.zld + 2 * c;
      if (g >= 0) {
        cp_async16(dst, Z64 + (int64_t)g * P + 2 * c);
      } else {
        dst[0] = 0.0;
        dst[1] = 0.0;
      }
    }
    cp_async_commit();
  };

  int cur_leaf = -1;
  issue_tile(t_begin, 0);
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int b = (tile - t_begin) & 1;
    const int li = prefix_find(h.tpre, n_leaf_nodes, tile);
    const int v = leaf_nodes[li];
    const int comp = pv.leaf_index[v];
    const int r = pv.model_rank[comp];
    cp_async_wait_all();
    __syncthreads();  // tile rows landed; previous tile's compute finished
    if (tile + 1 < t_end) issue_tile(tile + 1, b ^ 1);
    if (comp != cur_leaf) {
      const double* U = pv.model_basis + pv.model_off64[comp];
      for (int e = tid; e < geo.Pn * geo.R8; e += kThreads) {
        const int p = e / geo.R8, j = e - p * geo.R8;
        const double u = (p < P && j < r) ? U[(int64_t)p * r + j] : 0.0;
        Us[p * geo.uld + j] = u;
        UT[j * geo.utld + p] = u;
      }
      const double* shrink = pv.model_shrink + (int64_t)t * pv.model_cols_total + pv.model_col_off[comp];
      for (int j = tid; j < geo.R8; j += kThreads) sh[j] = j < r ? shrink[j] : 0.0;
      cur_leaf = comp;
      __syncthreads();
    }
    const double* Zs = b ? Zs1 : Zs0;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int m0 = warp * 8;
    // ---- phase 1: C[m0..m0+7][0..R8) = Z . U
    {
      double acc[kMaxR / 8][2];
      const int nt = geo.R8 / 8;
#pragma unroll
      for (int n = 0; n < kMaxR / 8; ++n) acc[n][0] = acc[n][1] = 0.0;
      for (int k0 = 0; k0 < P; k0 += 4) {
        const double a = Zs[(m0 + g4) * geo.zld + k0 + t4];
#pragma unroll
        for (int n = 0; n < kMaxR / 8; ++n)
          if (n < nt) dmma(acc[n], a, Us[(k0 + t4) * geo.uld + n * 8 + g4]);
      }
#pragma unroll
      for (int n = 0; n < kMaxR / 8; ++n)
        if (n < nt) {
          const int col = n * 8 + 2 * t4;
          Cs[(m0 + g4) * geo.cld + col] = acc[n][0] * sh[col];
          Cs[(m0 + g4) * geo.cld + col + 1] = acc[n][1] * sh[col + 1];
        }
    }
    __syncwarp();  // each warp only reads its own rows of Cs
    // ---- phase 2: Zhat[m0..m0+7][0..P) = C . U^T + gamma_tail Z
    {
      double acc[NT2][2];
#pragma unroll
      for (int n = 0; n < NT2; ++n) acc[n][0] = acc[n][1] = 0.0;
      for (int k0 = 0; k0 < geo.R8; k0 += 4) {
        const double a = Cs[(m0 + g4) * geo.cld + k0 + t4];
#pragma unroll
        for (int n = 0; n < NT2; ++n) dmma(acc[n], a, UT[(k0 + t4) * geo.utld + n * 8 + g4]);
      }
      const double gt = pv.model_gamma_tail[(int64_t)t * pv.K + comp];
      const int row = m0 + g4;
      const int gidx = h.rows[b][row];
      if (gidx >= 0) {
        double* out = Zhat + (int64_t)gidx * P;
#pragma unroll
        for (int n = 0; n < NT2; ++n) {
          const int col = n * 8 + 2 * t4;
          if (col < P) {
            double2 o;
            o.x = acc[n][0] + gt * Zs[row * geo.zld + col];
            o.y = acc[n][1] + gt * Zs[row * geo.zld + col + 1];
            *reinterpret_cast<double2*>(out + col) = o;
          }
        }
      }
    }
  }
}

}  // namespace wn

int wiener_dmma(Plan* p, int t, const double* Z64, double* Zhat, cudaStream_t st) {
  const int P = p->v.P;
  wn::Geo geo;
  geo.P = P;
  geo.Pn = (P + 7) / 8 * 8;
  auto ld = [](int n, int rem) { int v = n; while (v % 16 != rem) ++v; return v; };
  geo.zld = ld(P, 4);
  geo.R8 = (p->max_model_rank + 7) / 8 * 8;
  geo.uld = ld(geo.R8, 8);
  geo.utld = ld(geo.Pn, 8);
  geo.cld = ld(geo.R8, 4);
  const size_t smem = ((sizeof(wn::Head) + 127) & ~size_t(127)) +
                      sizeof(double) * (2 * (size_t)wn::kRows * geo.zld + (size_t)geo.Pn * geo.uld +
                                        (size_t)geo.R8 * geo.utld + (size_t)wn::kRows * geo.cld +
                                        geo.R8);
  const int nt2 = geo.Pn / 8;
  auto launch = [&](auto kernel) -> int {
    FEPLL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, wn::kThreads, smem);
    kernel<<<kSMs * std::max(1, per_sm), wn::kThreads, smem, st>>>(
        p->v, t, p->d_leaf_nodes, p->n_leaf_nodes, p->rs.cnt, p->rs.off, p->rs.leafseg, Z64, Zhat,
        geo);
    FEPLL_LAUNCH();
    return kOk;
  };
  switch (nt2) {
    case 1: return launch(wn::wiener_dmma_kernel<1>);
    case 2: return launch(wn::wiener_dmma_kernel<2>);
    case 4: return launch(wn::wiener_dmma_kernel<4>);
    case 5: return launch(wn::wiener_dmma_kernel<5>);
    case 7: return launch(wn::wiener_dmma_kernel<7>);
    case 8: return launch(wn::wiener_dmma_kernel<8>);
    case 11: return launch(wn::wiener_dmma_kernel<11>);
    case 13: return launch(wn::wiener_dmma_kernel<13>);
    case 16: return launch(wn::wiener_dmma_kernel<16>);
    default: break;
  }
  set_error("wiener: unsupported patch size for the DMMA kernel");
  return kDataError;
}

bool wiener_dmma_supported(const Plan* p) {
  const int P = p->v.P;
  const int nt2 = (P + 7) / 8;
  const bool nt_ok = nt2 == 1 || nt2 == 2 || nt2 == 4 || nt2 == 5 || nt2 == 7 || nt2 == 8 ||
                     nt2 == 11 || nt2 == 13 || nt2 == 16;
  return P % 4 == 0 && P <= wn::kMaxP && p->max_model_rank <= wn::kMaxR && nt_ok;
}

}  // namespace fepll
