// Shared tcgen05 scoring epilogue: one thread = one patch row (TMEM lane).
//
// For every child c of the tile's node (pkg/src/fepll/tree.py:417-425) the
// child's columns start on a 16-column boundary (plan.py tc_images), so the
// thread streams them in 16-column TMEM chunks and accumulates
// s_c = sum_j c_j^2 w_j and e_c = sum_j |c_j w_j| in FP32.
// score_c = const_c + ||z||^2 / nu_tail_c + s_c (FP64, gmm.py:335-338; the
// division is a multiplication by the FP64 reciprocal, a 1-ulp change
// covered by the bound's relative slack).
//
// Certification: the 3xTF32 projection (three FP32-accumulated tcgen05
// passes) is within 2^-18 ||z|| of the exact coefficient, and the FP32
// accumulation adds <= 64 * 2^-24 * sum|c^2 w| <= 2^-18 ||z|| sum|c w|;
// err_c = guard * ||z|| * e_c + 2^-40 |score_c| with guard = 2^-16 covers
// both with margin.  The argmin is certified when every other child
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
    E.col[tid] = pv.tc_child_col[v];
    E.chunks[tid] = (pv.node_rank[v] + 15) >> 4;
    E.bfs[tid] = v;
  }
}

// Returns the best child index; *flagged when the decision is not certified.
// d_acc: TMEM address (lane field set) of the tile's accumulator.
__device__ __forceinline__ int epi_score_row(const EpiChild& E, int nk, uint32_t d_acc,
                                             double sqv, double guard, bool* flagged) {
  const double zn = (double)sqrtf((float)sqv) * (1.0 + 1e-6);
  double best = INFINITY, best_err = 0.0, m1 = INFINITY, m2 = INFINITY;
  int bi = 0, i1 = -1;
  for (int ci = 0; ci < nk; ++ci) {
    const int c0 = E.col[ci];
    float s0 = 0.f, s1 = 0.f, e0 = 0.f, e1 = 0.f;
    for (int q = 0; q < E.chunks[ci]; ++q) {
      uint32_t ra[16];
      tmem_ld16(d_acc + c0 + 16 * q, ra);
      tc::tmem_ld_wait();
      const float* w = E.w + c0 + 16 * q;
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const float ca = __uint_as_float(ra[j]);
        const float cb = __uint_as_float(ra[j + 1]);
        const float wa = ca * w[j], wb = cb * w[j + 1];
        s0 = fmaf(wa, ca, s0);
        s1 = fmaf(wb, cb, s1);
        e0 += fabsf(wa);
        e1 += fabsf(wb);
      }
    }
    const double sc = E.cconst[ci] + sqv * E.cinvnut[ci] + ((double)s0 + (double)s1);
    const double er = guard * zn * ((double)e0 + (double)e1) + 0x1p-40 * fabs(sc);
    if (sc < best) { best = sc; bi = ci; best_err = er; }
    const double lo = sc - er;
    if (lo < m1) { m2 = m1; m1 = lo; i1 = ci; }
    else if (lo < m2) { m2 = lo; }
  }
  const double other = (i1 == bi) ? m2 : m1;
  *flagged = !(other > best + best_err) || !isfinite(best);
  return bi;
}

}  // namespace fepll
