// Shared tcgen05 scoring epilogue: one thread = one patch row (TMEM lane).
//
// For every child c of the tile's node (pkg/src/fepll/tree.py:417-425) the
// child's columns start on a 16-column boundary (plan.py tc_images), so the
// thread streams them in 16-column TMEM chunks.  The B columns carry
// sqrt(-w_j) (w = sq_weight <= 0 at the iteration's beta), so the
// accumulators hold c'_j = c_j sqrt(-w_j) and s_c = sum_j c_j^2 w_j =
// -sum_j c'_j^2: one packed FP32x2 FMA (FFMA2) per two columns.
// score_c = const_c + ||z||^2 / nu_tail_c + s_c (FP64, gmm.py:335-338; the
// division is a multiplication by the FP64 reciprocal fused with the add, a
// few-ulp change covered by the bound's 2^-40 relative slack).
//
// Certification: the 3xTF32 projection (three FP32-accumulated tcgen05
// passes) is within gamma = 2^-18 ||z|| ||b_j|| of the exact c'_j (b_j the
// scaled column, ||b_j|| = sqrt|w_j|), so
// |d s_c| <= 2 gamma sum_j |c'_j| sqrt|w_j| ||z|| = 2^-17 ||z|| sum_j |c_j w_j|
// <= 2^-17 ||z||^2 ||w_c|| (Cauchy-Schwarz, ||c|| <= ||z||); the FP32
// accumulation adds <= 65 * 2^-24 * sum_j c'_j^2 <= 2^-18 ||z||^2 ||w_c||.
// err_c = guard * ||z||^2 * ||w_c|| + 2^-40 |score_c| with guard = 2^-16
// covers both.  The argmin is certified when every other child
// satisfies score_c - err_c > score_best + err_best; otherwise the caller
// queues the patch for exact FP64 re-scoring.
#pragma once
#include "common.cuh"
#include "tc.cuh"

namespace fepll {

constexpr double kDefaultGuard = 1.52587890625e-05;  // 2^-16

struct EpiChild {
  double cconst[kMaxChildren];
  double cinvnut[kMaxChildren];   // 1 / nu_tail
  double wnorm[kMaxChildren];     // ||w_c|| of the FP32 column weights
  int32_t col[kMaxChildren];     // 16-aligned first column in the node's image
  int32_t chunks[kMaxChildren];  // ceil(rank / 16)
  int32_t bfs[kMaxChildren];
  float w[256];                  // per-column FP32 weights of the node image
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Load the child tables of node u at iteration t (cooperative, nthreads).
__device__ __forceinline__ void epi_load_node(const PlanView& pv, int t, int u, EpiChild& E,
                                              int tid, int nthreads) {
  const int nk = pv.child_count[u];
  const int npad = pv.tc_npad[u];
  const float* w = pv.tc_w + (int64_t)t * pv.tc_w_cols + pv.tc_w_off[u];
  for (int j = tid; j < npad; j += nthreads) E.w[j] = w[j];
  if (tid < nk) {
    const int v = pv.child_list[pv.child_start[u] + tid];
    const int64_t ti = (int64_t)t * pv.n_nodes + v;
    E.cconst[tid] = pv.node_const[ti];
    E.cinvnut[tid] = 1.0 / pv.node_nu_tail[ti];
    const float* wc = w + pv.tc_child_col[v];
    double n2 = 0.0;
    for (int j = 0; j < pv.node_rank[v]; ++j) n2 += (double)wc[j] * (double)wc[j];
    E.wnorm[tid] = sqrt(n2);
    E.col[tid] = pv.tc_child_col[v];
    E.chunks[tid] = (pv.node_rank[v] + 15) >> 4;
    E.bfs[tid] = v;
  }
}

__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Running certified argmin over children scored chunk by chunk (wide nodes
// stream their columns through TMEM in several chunks; a normal node is one
// chunk).  m1/m2: the two smallest lower bounds score - err seen so far.
struct EpiRun {
  double best = INFINITY, best_err = 0.0, m1 = INFINITY, m2 = INFINITY;
  int bi = 0, i1 = -1;
};

// Score children 0..nk-1 of the chunk in E (TMEM columns E.col[ci] of
// d_acc); k_base: index of E's first child among the node's children.
__device__ __forceinline__ void epi_run_chunk(const EpiChild& E, int nk, int k_base, uint32_t d_acc,
                                              double sqv, double guard, EpiRun& R) {
  const double gs = guard * sqv;  // per-row part of the bound
  for (int ci = 0; ci < nk; ++ci) {
    const int c0 = E.col[ci];
    uint64_t s2 = 0;  // two FP32 partial sums
    for (int q = 0; q < E.chunks[ci]; ++q) {
      uint32_t ra[16];
      tmem_ld16(d_acc + c0 + 16 * q, ra);
      tc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t c2 = (uint64_t)ra[2 * j] | ((uint64_t)ra[2 * j + 1] << 32);
        s2 = f2_fma(c2, c2, s2);
      }
    }
    // the two FP32 partial sums meet in FP32 (one more rounding, inside the
    // accumulation budget), the score and its bound in fused FP64 ops
    const float sf = __uint_as_float((uint32_t)s2) + __uint_as_float((uint32_t)(s2 >> 32));
    // the B columns carry sqrt(-w_j) (plan.py tc_images): sum_j c_j^2 w_j = -sum_j c'_j^2
    const double sc = fma(sqv, E.cinvnut[ci], E.cconst[ci]) - (double)sf;
    const double er = fma(0x1p-40, fabs(sc), gs * E.wnorm[ci]);
    const int k = k_base + ci;
    if (sc < R.best) { R.best = sc; R.bi = k; R.best_err = er; }
    const double lo = sc - er;
    if (lo < R.m1) { R.m2 = R.m1; R.m1 = lo; R.i1 = k; }
    else if (lo < R.m2) { R.m2 = lo; }
  }
}

// certified iff every other child's lower bound clears the best's upper one
__device__ __forceinline__ bool epi_run_flagged(const EpiRun& R) {
  const double other = (R.i1 == R.bi) ? R.m2 : R.m1;
  return !(other > R.best + R.best_err) || !isfinite(R.best);
}

// Returns the best child index; *flagged when the decision is not certified.
// d_acc: TMEM address (lane field set) of the tile's accumulator.
__device__ __forceinline__ int epi_score_row(const EpiChild& E, int nk, uint32_t d_acc,
                                             double sqv, double guard, bool* flagged) {
  EpiRun R;
  epi_run_chunk(E, nk, 0, d_acc, sqv, guard, R);
  *flagged = epi_run_flagged(R);
  return R.bi;
}

}  // namespace fepll
