// Kernel (e) for the non-pixel operators + the per-restore operator setup.
//
// Restates pkg/src/fepll/operators.py on the device, FP64 throughout (an
// FP32 solve flips tree decisions downstream):
//   apply / apply_adjoint / normal_apply   :200-235 (circular convolution as
//        a direct periodic stencil — the same linear map as the reference's
//        FFT product, to rounding; decimation keeps every d-th sample)
//   conjugate_gradient                      :242-266 (one cooperative kernel,
//        grid-wide barriers between phases, deterministic reductions)
//   solve_image_estimation                  :273-295 (FFT for convolution,
//        CG for decimation; pixel kinds are fused into aggregate.cu)
//   _power_iteration_l2sq                   :298-319 (cooperative kernel)
//   init_estimate                           :374-394 (FFT / CG with the
//        periodic Laplacian)
#include <algorithm>
#include <cmath>
#include <cooperative_groups.h>

#include "fft.cuh"

namespace cg = cooperative_groups;

namespace fepll {

// ------------------------------------------------------------------ FFT tables
int fft_dim_build(int n, FftDim* out, std::vector<void*>* owned) {
  FEPLL_REQUIRE(n >= 1 && n <= kFftMaxN, "fft: length out of range (1..4096)");
  std::vector<int> radix;
  int m = n;
  for (int p : {4, 2, 3, 5, 7}) {
    while (m % p == 0) { radix.push_back(p); m /= p; }
  }
  for (int p = 11; m > 1; p += 2) {
    while (m % p == 0) { radix.push_back(p); m /= p; }
  }
  FEPLL_REQUIRE((int)radix.size() <= kFftMaxStages, "fft: too many stages");
  for (int r : radix) FEPLL_REQUIRE(r <= kFftMaxRadix, "fft: prime factor above 64 unsupported");
  std::vector<double2> tw, root;
  FftDim d;
  d.n = n;
  d.stages = (int)radix.size();
  int Ns = 1;
  const double two_pi = 6.283185307179586476925286766559;
  for (int s = 0; s < d.stages; ++s) {
    const int R = radix[s];
    d.radix[s] = R;
    d.ns[s] = Ns;
    d.tw_off[s] = (int)tw.size();
    for (int jj = 0; jj < Ns; ++jj)
      for (int r = 0; r < R; ++r) {
        const double ang = -two_pi * (double)(r * jj) / (double)(Ns * R);
        tw.push_back(make_double2(std::cos(ang), std::sin(ang)));
      }
    d.root_off[s] = (int)root.size();
    for (int e = 0; e < R; ++e) {
      const double ang = -two_pi * (double)e / (double)R;
      root.push_back(make_double2(std::cos(ang), std::sin(ang)));
    }
    Ns *= R;
  }
  if (tw.empty()) tw.push_back(make_double2(1.0, 0.0));
  void* dt = nullptr;
  void* dr = nullptr;
  FEPLL_CUDA(cudaMalloc(&dt, sizeof(double2) * tw.size()));
  FEPLL_CUDA(cudaMalloc(&dr, sizeof(double2) * root.size()));
  owned->push_back(dt);
  owned->push_back(dr);
  FEPLL_CUDA(cudaMemcpy(dt, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
  FEPLL_CUDA(cudaMemcpy(dr, root.data(), sizeof(double2) * root.size(), cudaMemcpyHostToDevice));
  d.tw = static_cast<const double2*>(dt);
  d.root = static_cast<const double2*>(dr);
  *out = d;
  return kOk;
}

// ------------------------------------------------------------------ op plan
enum OpKind { kIdentity = 0, kConvolution = 1, kMask = 2, kGain = 3, kDecimate = 4 };

struct OpView {
  int kind, H, W, Ho, Wo, d;  // d = decimation factor (1 otherwise)
  int kh, kw;
  const double* taps;         // [kh][kw]
  const double* diag;         // [H][W] diag(A^T A) for mask/gain
  const double* pmap;         // [H][W] mask (0/1) or gain
  const double2* khat;        // [H][W] DFT of the centred kernel (convolution)
  const double* kabs2;        // [H][W] |khat|^2
  const double* lsym;         // [H][W] periodic Laplacian symbol
};

struct OpPlan {
  OpView v{};
  FftDim fr, fc;              // row (length W) and column (length H) transforms
  std::vector<void*> owned;
  double2* work = nullptr;    // H x W complex scratch
  double* low = nullptr;      // Ho x Wo scratch (decimate)
  double* r = nullptr;        // CG vectors
  double* p = nullptr;
  double* p2 = nullptr;       // CG direction ping-pong
  double* ap = nullptr;
  double* partial = nullptr;  // per-block partial sums (4 per block: two buffers of up to 2)
  double* scal = nullptr;     // device scalars
  int coop_blocks = 0;
};

// ------------------------------------------------------------------ stencils
__device__ __forceinline__ int wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// element sources for the stencils: a vector, or the CG direction formed
// on the fly, p = r + beta p_old (the same FMA the update itself uses)
struct VecSrc {
  const double* x;
  __device__ __forceinline__ double operator()(int64_t i) const { return x[i]; }
};
struct DirSrc {
  const double* r;
  const double* pold;
  double beta;
  __device__ __forceinline__ double operator()(int64_t i) const { return fma(beta, pold[i], r[i]); }
};

// (conv x)[p] = sum_ab k[a][b] x[p - (a - ch, b - cw)]   (operators.py:196-197 with kernel_ft)
template <class Src>
__device__ __forceinline__ double conv_at_src(const OpView& o, const Src& x, int r, int c) {
  const int ch = o.kh / 2, cw = o.kw / 2;
  double s = 0.0;
  for (int a = 0; a < o.kh; ++a) {
    const int64_t row = (int64_t)wrap(r - a + ch, o.H) * o.W;
    for (int b = 0; b < o.kw; ++b) s = fma(o.taps[a * o.kw + b], x(row + wrap(c - b + cw, o.W)), s);
  }
  return s;
}
__device__ __forceinline__ double conv_at(const OpView& o, const double* x, int r, int c) {
  return conv_at_src(o, VecSrc{x}, r, c);
}

// adjoint: correlation with the kernel (conj khat), over the zero-filled
// up-sampled input when decimating
__device__ __forceinline__ double corr_at(const OpView& o, const double* y, int r, int c) {
  const int ch = o.kh / 2, cw = o.kw / 2;
  double s = 0.0;
  for (int a = 0; a < o.kh; ++a) {
    const int rr = wrap(r + a - ch, o.H);
    if (rr % o.d) continue;
    const double* row = y + (int64_t)(rr / o.d) * o.Wo;
    for (int b = 0; b < o.kw; ++b) {
      const int cc = wrap(c + b - cw, o.W);
      if (cc % o.d) continue;
      s = fma(o.taps[a * o.kw + b], row[cc / o.d], s);
    }
  }
  return s;
}

template <class Src>
__device__ __forceinline__ double lap_at_src(const Src& x, int r, int c, int H, int W) {
  const int64_t row = (int64_t)r * W;
  return 4.0 * x(row + c) - x((int64_t)wrap(r - 1, H) * W + c) - x((int64_t)wrap(r + 1, H) * W + c) -
         x(row + wrap(c - 1, W)) - x(row + wrap(c + 1, W));
}
__device__ __forceinline__ double lap_at(const double* x, int r, int c, int H, int W) {
  return lap_at_src(VecSrc{x}, r, c, H, W);
}

// ------------------------------------------------------------------ reductions
// deterministic grid reduction: fixed per-thread order, fixed block tree,
// every block sums the block partials in index order.
template <int NV>
__device__ inline void block_reduce_store(double (&v)[NV], double* partial, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double x = v[i];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[w * NV + i] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k * NV + i];
      partial[blockIdx.x * NV + i] = s;
    }
  }
  __syncthreads();
}

// every block: the sum of the block partials, warp 0 in a fixed order (lane
// l sums blocks l, l + 32, ... in turn, then a fixed shuffle tree) — one
// round of independent loads instead of a serial walk over the blocks
template <int NV>
__device__ inline void grid_total(const double* partial, double (&out)[NV], double* red) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) s += partial[b * NV + i];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[i] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) out[i] = red[i];
  __syncthreads();
}

// ------------------------------------------------------------------ normal op
// y = (A^T A) x + shift * x + lapc * L x, two phases when A has a stencil:
// phase A writes low = conv/decimate(x) (Ho x Wo), phase B the rest.
struct NormalArgs {
  OpView o;
  double shift, lapc;
};

template <class Src>
__device__ inline void normal_phase_a_src(const NormalArgs& n, const Src& x, double* low,
                                          int64_t gtid, int64_t gstride) {
  const OpView& o = n.o;
  if (o.kind != kConvolution && o.kind != kDecimate) return;
  const int64_t total = (int64_t)o.Ho * o.Wo;
  for (int64_t i = gtid; i < total; i += gstride) {
    const int r = (int)(i / o.Wo), c = (int)(i - (int64_t)r * o.Wo);
    low[i] = conv_at_src(o, x, r * o.d, c * o.d);
  }
}
__device__ inline void normal_phase_a(const NormalArgs& n, const double* x, double* low,
                                      int64_t gtid, int64_t gstride) {
  normal_phase_a_src(n, VecSrc{x}, low, gtid, gstride);
}

// xi = the source's element i (the caller has it at hand)
template <class Src>
__device__ inline double normal_phase_b_src(const NormalArgs& n, const Src& x, double xi,
                                            const double* low, int r, int c) {
  const OpView& o = n.o;
  const int64_t i = (int64_t)r * o.W + c;
  double y;
  switch (o.kind) {
    case kIdentity: y = xi; break;
    case kMask:
    case kGain: y = o.diag[i] * xi; break;
    default: y = corr_at(o, low, r, c); break;
  }
  if (n.shift != 0.0) y += n.shift * xi;
  if (n.lapc != 0.0) y += n.lapc * lap_at_src(x, r, c, o.H, o.W);
  return y;
}
__device__ inline double normal_phase_b(const NormalArgs& n, const double* x, const double* low,
                                        int r, int c) {
  return normal_phase_b_src(n, VecSrc{x}, x[(int64_t)r * n.o.W + c], low, r, c);
}

// ------------------------------------------------------------------ CG kernel
struct CgArgs {
  NormalArgs nrm;
  const double* rhs;
  double* x;         // in: x0, out: solution
  double* r;
  double* p;         // direction, ping-pong with p2
  double* p2;
  double* ap;
  double* low;
  double* partial;
  double* out;       // [0] iterations, [1] residual, [2] converged, [3] finite
  int32_t* status;   // optional: bit 2 set when the solution is non-finite
  double tol;
  int maxit;
};

// Standard CG (operators.py:242-266) with three grid barriers per
// iteration: the direction p_k = r_k + beta p_{k-1} is not written before
// the next operator application — the stencils form it on the fly from r
// and p_{k-1} (DirSrc, the update's own FMA) while each thread stores its
// own elements into the other p buffer — and the two dot products use
// separate partial buffers.  Iterates: those of the reference recursion.
__global__ void __launch_bounds__(256) cg_kernel(CgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[64];
  const OpView& o = a.nrm.o;
  const int64_t N = (int64_t)o.H * o.W;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  double* partA = a.partial;                  // <p, Ap>, and the setup sums
  double* partB = a.partial + 2 * gridDim.x;  // <r, r>
  double v1[1], t1[1];
  // rn = ||rhs||
  v1[0] = 0.0;
  for (int64_t i = gtid; i < N; i += gs) v1[0] = fma(a.rhs[i], a.rhs[i], v1[0]);
  block_reduce_store(v1, partA, red);
  grid.sync();
  grid_total<1>(partA, t1, red);
  const double rn = sqrt(t1[0]);
  if (rn == 0.0) {
    for (int64_t i = gtid; i < N; i += gs) a.x[i] = 0.0;
    if (gtid == 0) { a.out[0] = 0; a.out[1] = 0; a.out[2] = 1; a.out[3] = 1; }
    return;
  }
  // r = rhs - op(x); rs = <r,r>  (p_0 = r is formed on the fly)
  normal_phase_a(a.nrm, a.x, a.low, gtid, gs);
  grid.sync();
  v1[0] = 0.0;
  for (int64_t i = gtid; i < N; i += gs) {
    const int rr = (int)(i / o.W), cc = (int)(i - (int64_t)rr * o.W);
    const double ri = a.rhs[i] - normal_phase_b(a.nrm, a.x, a.low, rr, cc);
    a.r[i] = ri;
    v1[0] = fma(ri, ri, v1[0]);
  }
  block_reduce_store(v1, partB, red);
  grid.sync();
  grid_total<1>(partB, t1, red);
  double rs = t1[0];
  double beta = 0.0;
  double* pold = a.p;   // p_{k-1} (unused while beta is 0 on the first pass)
  double* pnew = a.p2;  // receives p_k
  int it = 0;
  for (it = 1; it <= a.maxit; ++it) {
    if (sqrt(rs) / rn <= a.tol) { --it; break; }
    // low = conv(p_k) with p_k = r + beta p_{k-1} on the fly
    if (it == 1)
      normal_phase_a(a.nrm, a.r, a.low, gtid, gs);
    else
      normal_phase_a_src(a.nrm, DirSrc{a.r, pold, beta}, a.low, gtid, gs);
    grid.sync();
    v1[0] = 0.0;
    for (int64_t i = gtid; i < N; i += gs) {
      const int rr = (int)(i / o.W), cc = (int)(i - (int64_t)rr * o.W);
      const double pi = it == 1 ? a.r[i] : fma(beta, pold[i], a.r[i]);
      const double api = it == 1 ? normal_phase_b_src(a.nrm, VecSrc{a.r}, pi, a.low, rr, cc)
                                 : normal_phase_b_src(a.nrm, DirSrc{a.r, pold, beta}, pi, a.low, rr, cc);
      pnew[i] = pi;
      a.ap[i] = api;
      v1[0] = fma(pi, api, v1[0]);
    }
    block_reduce_store(v1, partA, red);
    grid.sync();  // partials ready; every stencil read of r and p_{k-1} is done
    grid_total<1>(partA, t1, red);
    const double alpha = rs / t1[0];
    v1[0] = 0.0;
    for (int64_t i = gtid; i < N; i += gs) {
      a.x[i] += alpha * pnew[i];
      const double ri = a.r[i] - alpha * a.ap[i];
      a.r[i] = ri;
      v1[0] = fma(ri, ri, v1[0]);
    }
    block_reduce_store(v1, partB, red);
    grid.sync();  // r_{k+1} and p_k complete for the next iteration's stencils
    grid_total<1>(partB, t1, red);
    const double rs_new = t1[0];
    beta = rs_new / rs;
    rs = rs_new;
    double* tp = pold;
    pold = pnew;
    pnew = tp;
  }
  if (it > a.maxit) it = a.maxit;
  // residual = ||rhs - op(x)|| / rn
  grid.sync();
  normal_phase_a(a.nrm, a.x, a.low, gtid, gs);
  grid.sync();
  double v2[2] = {0.0, 0.0}, t2[2];
  for (int64_t i = gtid; i < N; i += gs) {
    const int rr = (int)(i / o.W), cc = (int)(i - (int64_t)rr * o.W);
    const double d = a.rhs[i] - normal_phase_b(a.nrm, a.x, a.low, rr, cc);
    v2[0] = fma(d, d, v2[0]);
    if (!isfinite(a.x[i])) v2[1] += 1.0;
  }
  block_reduce_store(v2, partA, red);
  grid.sync();
  grid_total<2>(partA, t2, red);
  if (gtid == 0) {
    const double res = sqrt(t2[0]) / rn;
    a.out[0] = it;
    a.out[1] = res;
    a.out[2] = res <= a.tol ? 1.0 : 0.0;
    a.out[3] = t2[1] == 0.0 ? 1.0 : 0.0;
    // sticky across the calls sharing one status word (out[] is per call)
    if (a.status && t2[1] != 0.0) atomicOr(a.status, 2);
  }
}

// ------------------------------------------------------------------ power iteration
struct PowerArgs {
  NormalArgs nrm;
  double* v;        // in: start vector (unnormalised), scratch
  double* w;
  double* low;
  double* partial;
  double* out;      // [0] lambda
  int iters;
  double tol;
};

__global__ void __launch_bounds__(256) power_kernel(PowerArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[64];
  const OpView& o = a.nrm.o;
  const int64_t N = (int64_t)o.H * o.W;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  double v1[1], t1[1], v2[2], t2[2];
  // v /= ||v||
  v1[0] = 0.0;
  for (int64_t i = gtid; i < N; i += gs) v1[0] = fma(a.v[i], a.v[i], v1[0]);
  block_reduce_store(v1, a.partial, red);
  grid.sync();
  grid_total<1>(a.partial, t1, red);
  const double n0 = sqrt(t1[0]);
  for (int64_t i = gtid; i < N; i += gs) a.v[i] /= n0;
  double prev = 0.0, lam = 0.0;
  for (int k = 0; k < a.iters; ++k) {
    grid.sync();
    normal_phase_a(a.nrm, a.v, a.low, gtid, gs);
    grid.sync();
    v2[0] = v2[1] = 0.0;
    for (int64_t i = gtid; i < N; i += gs) {
      const int rr = (int)(i / o.W), cc = (int)(i - (int64_t)rr * o.W);
      const double wi = normal_phase_b(a.nrm, a.v, a.low, rr, cc);
      a.w[i] = wi;
      v2[0] = fma(a.v[i], wi, v2[0]);
      v2[1] = fma(wi, wi, v2[1]);
    }
    block_reduce_store(v2, a.partial, red);
    grid.sync();
    grid_total<2>(a.partial, t2, red);
    lam = t2[0];
    const double nrm = sqrt(t2[1]);
    if (nrm == 0.0) { lam = 0.0; break; }
    for (int64_t i = gtid; i < N; i += gs) a.v[i] = a.w[i] / nrm;
    if (prev > 0.0 && fabs(lam - prev) <= a.tol * fabs(lam)) break;
    prev = lam;
  }
  if (gtid == 0) a.out[0] = lam;
}

// ------------------------------------------------------------------ FFT kernels
// rows: forward transform of every row (real or complex input) into work
__global__ void fft_rows_fwd(FftDim fd, const double* re, const double2* cin, double2* work,
                             int W) {
  extern __shared__ double2 sm[];
  double2* d0 = sm;
  double2* d1 = sm + fd.n;
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < W; c += blockDim.x)
    d0[c] = re ? make_double2(re[(int64_t)r * W + c], 0.0) : cin[(int64_t)r * W + c];
  __syncthreads();
  double2* out = fft_smem(fd, d0, d1);
  for (int c = threadIdx.x; c < W; c += blockDim.x) work[(int64_t)r * W + c] = out[c];
}

enum FilterMode {
  kFilterNone = 0,        // forward only: keep the spectrum
  kFilterSolve = 1,       // X / (|khat|^2 + s)            (operators.py:288-292)
  kFilterAdjoint = 2,     // X * conj(khat)                 (operators.py:222-223)
  kFilterInit = 3,        // X * conj(ft) / (|ft|^2 + c Ls) (operators.py:382-389)
};

// columns: forward transform, spectral filter, inverse transform (conj trick)
__global__ void fft_cols_filter(FftDim fd, double2* work, int H, int W, OpView o, int mode,
                                double s) {
  extern __shared__ double2 sm[];
  double2* d0 = sm;
  double2* d1 = sm + fd.n;
  const int c = blockIdx.x;
  for (int r = threadIdx.x; r < H; r += blockDim.x) d0[r] = work[(int64_t)r * W + c];
  __syncthreads();
  double2* spec = fft_smem(fd, d0, d1);
  double2* other = spec == d0 ? d1 : d0;
  if (mode == kFilterNone) {
    for (int r = threadIdx.x; r < H; r += blockDim.x) work[(int64_t)r * W + c] = spec[r];
    return;
  }
  for (int r = threadIdx.x; r < H; r += blockDim.x) {
    const int64_t f = (int64_t)r * W + c;
    double2 X = spec[r];
    double2 Y;
    if (mode == kFilterSolve) {
      const double den = o.kabs2[f] + s;
      Y = make_double2(X.x / den, X.y / den);
    } else if (mode == kFilterAdjoint) {
      const double2 k = o.khat[f];
      Y = cmul(X, make_double2(k.x, -k.y));
    } else {
      double2 k = o.khat ? o.khat[f] : make_double2(1.0, 0.0);
      const double k2 = o.khat ? o.kabs2[f] : 1.0;
      double den = k2 + s * o.lsym[f];
      if (f == 0 && den == 0.0) den = 1.0;
      const double2 num = cmul(make_double2(k.x, -k.y), X);
      Y = make_double2(num.x / den, num.y / den);
    }
    other[r] = make_double2(Y.x, -Y.y);  // conjugate for the inverse
  }
  __syncthreads();
  double2* back = fft_smem(fd, other, spec);
  for (int r = threadIdx.x; r < H; r += blockDim.x) work[(int64_t)r * W + c] = back[r];
}

// rows: inverse transform (input conjugated by the column pass), real part / (H W)
__global__ void fft_rows_inv_real(FftDim fd, const double2* work, double* out, int W, double scale,
                                  int32_t* status) {
  extern __shared__ double2 sm[];
  double2* d0 = sm;
  double2* d1 = sm + fd.n;
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < W; c += blockDim.x) d0[c] = work[(int64_t)r * W + c];
  __syncthreads();
  double2* res = fft_smem(fd, d0, d1);
  // conj(fft(conj(Y))) = N ifft(Y): the real part is unaffected by the outer conj
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    const double v = res[c].x * scale;
    out[(int64_t)r * W + c] = v;
    if (status && !isfinite(v)) atomicOr(status, 2);
  }
}

__global__ void pixel_adjoint_kernel(const double* y, const double* pmap, double* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = pmap ? pmap[i] * y[i] : y[i];
}

__global__ void decimate_adjoint_kernel(OpView o, const double* y, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)o.H * o.W) return;
  const int r = (int)(i / o.W), c = (int)(i - (int64_t)r * o.W);
  out[i] = corr_at(o, y, r, c);
}

__global__ void spectrum_abs2(const double2* k, double* a2, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a2[i] = k[i].x * k[i].x + k[i].y * k[i].y;
}

__global__ void normal_a_kernel(NormalArgs n, const double* x, double* low) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  normal_phase_a(n, x, low, i, (int64_t)gridDim.x * blockDim.x);
}

__global__ void normal_b_kernel(NormalArgs n, const double* x, const double* low, double* y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n.o.H * n.o.W) return;
  const int r = (int)(i / n.o.W), c = (int)(i - (int64_t)r * n.o.W);
  y[i] = normal_phase_b(n, x, low, r, c);
}

// ------------------------------------------------------------------ host glue
static size_t fft_smem(int n) { return 2 * sizeof(double2) * (size_t)n; }

static int fft_filter_2d(OpPlan* p, const double* re_in, int mode, double s, double* out,
                         int32_t* status, cudaStream_t st) {
  const int H = p->v.H, W = p->v.W;
  fft_rows_fwd<<<H, 256, fft_smem(W), st>>>(p->fr, re_in, nullptr, p->work, W);
  FEPLL_LAUNCH();
  fft_cols_filter<<<W, 256, fft_smem(H), st>>>(p->fc, p->work, H, W, p->v, mode, s);
  FEPLL_LAUNCH();
  if (mode == kFilterNone) return kOk;
  fft_rows_inv_real<<<H, 256, fft_smem(W), st>>>(p->fr, p->work, out, W, 1.0 / ((double)H * W),
                                                 status);
  FEPLL_LAUNCH();
  return kOk;
}

template <typename T>
static int dalloc(OpPlan* p, T** ptr, size_t count) {
  void* m = nullptr;
  FEPLL_CUDA(cudaMalloc(&m, sizeof(T) * std::max<size_t>(count, 1)));
  p->owned.push_back(m);
  *ptr = static_cast<T*>(m);
  return kOk;
}

#define DALLOC(ptr, count)                 \
  do {                                     \
    int _rc = dalloc(p, &(ptr), (count));  \
    if (_rc) return _rc;                   \
  } while (0)

static int coop_launch(const void* fn, void* args, OpPlan* p, cudaStream_t st) {
  void* kargs[] = {args};
  FEPLL_CUDA(cudaLaunchCooperativeKernel(fn, dim3(p->coop_blocks), dim3(256), kargs, 0, st));
  count_launch();
  return kOk;
}

}  // namespace fepll

using namespace fepll;

extern "C" {

int fepll_op_create(int32_t kind, int32_t H, int32_t W, int32_t factor, const double* taps,
                    int32_t kh, int32_t kw, const double* pixel_map, void** out) {
  FEPLL_REQUIRE(out != nullptr && H > 0 && W > 0, "op_create: bad arguments");
  FEPLL_REQUIRE(kind >= kIdentity && kind <= kDecimate, "op_create: unknown operator kind");
  OpPlan* p = new OpPlan();
  OpView& v = p->v;
  v.kind = kind;
  v.H = H;
  v.W = W;
  v.d = kind == kDecimate ? factor : 1;
  if (kind == kDecimate) {
    if (factor < 2 || H % factor || W % factor) {
      delete p;
      set_error("op_create: dims not divisible by the decimation factor");
      return kDataError;
    }
  }
  v.Ho = H / v.d;
  v.Wo = W / v.d;
  const int64_t N = (int64_t)H * W;
  if (kind == kConvolution || kind == kDecimate) {
    if (!taps || kh < 1 || kw < 1 || kh % 2 == 0 || kw % 2 == 0 || kh > H || kw > W) {
      delete p;
      set_error("op_create: kernel must be 2-D with odd sides and fit the image");
      return kDataError;
    }
    double* dt;
    DALLOC(dt, (size_t)kh * kw);
    FEPLL_CUDA(cudaMemcpy(dt, taps, sizeof(double) * kh * kw, cudaMemcpyHostToDevice));
    v.taps = dt;
    v.kh = kh;
    v.kw = kw;
  }
  if (kind == kMask || kind == kGain) {
    FEPLL_REQUIRE(pixel_map != nullptr, "op_create: pixel map required");
    std::vector<double> diag(N);
    for (int64_t i = 0; i < N; ++i)
      diag[i] = kind == kMask ? pixel_map[i] : pixel_map[i] * pixel_map[i];
    double *dm, *dd;
    DALLOC(dm, N);
    DALLOC(dd, N);
    FEPLL_CUDA(cudaMemcpy(dm, pixel_map, sizeof(double) * N, cudaMemcpyHostToDevice));
    FEPLL_CUDA(cudaMemcpy(dd, diag.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
    v.pmap = dm;
    v.diag = dd;
  }
  // FFT support (convolution kind, and the Laplacian-regularised init of identity)
  if (kind == kConvolution || kind == kIdentity) {
    if (H <= kFftMaxN && W <= kFftMaxN) {
      int rc = fft_dim_build(W, &p->fr, &p->owned);
      if (!rc) rc = fft_dim_build(H, &p->fc, &p->owned);
      if (rc) { delete p; return rc; }
      DALLOC(p->work, N);
      double* ls;
      DALLOC(ls, N);
      std::vector<double> lsh(N);
      const double two_pi = 6.283185307179586476925286766559;
      for (int r = 0; r < H; ++r) {
        // np.fft.fftfreq(H)[r] = r/H for r < ceil(H/2), else (r-H)/H
        const double fr = (r < (H + 1) / 2 ? r : r - H) / (double)H;
        for (int c = 0; c < W; ++c) {
          const double fc = (c < (W + 1) / 2 ? c : c - W) / (double)W;
          lsh[(int64_t)r * W + c] = 4.0 - 2.0 * std::cos(two_pi * fr) - 2.0 * std::cos(two_pi * fc);
        }
      }
      FEPLL_CUDA(cudaMemcpy(ls, lsh.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
      v.lsym = ls;
    }
  }
  if (kind == kConvolution) {
    FEPLL_REQUIRE(p->work != nullptr, "op_create: image too large for the FFT (<= 4096 per side)");
    // kernel_ft (operators.py:91-100): zero-pad, roll by -(k//2), fft2
    std::vector<double> pad(N, 0.0);
    for (int a = 0; a < kh; ++a)
      for (int b = 0; b < kw; ++b) {
        const int r = ((a - kh / 2) % H + H) % H, c = ((b - kw / 2) % W + W) % W;
        pad[(int64_t)r * W + c] = taps[a * kw + b];
      }
    double* dpad;
    DALLOC(dpad, N);
    FEPLL_CUDA(cudaMemcpy(dpad, pad.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
    double2* kh2;
    double* a2;
    DALLOC(kh2, N);
    DALLOC(a2, N);
    int rc = fft_filter_2d(p, dpad, kFilterNone, 0.0, nullptr, nullptr, 0);
    if (rc) { delete p; return rc; }
    FEPLL_CUDA(cudaMemcpy(kh2, p->work, sizeof(double2) * N, cudaMemcpyDeviceToDevice));
    spectrum_abs2<<<(unsigned)((N + 255) / 256), 256>>>(kh2, a2, N);
    FEPLL_CUDA(cudaDeviceSynchronize());
    v.khat = kh2;
    v.kabs2 = a2;
  }
  // CG / power-iteration scratch
  DALLOC(p->r, N);
  DALLOC(p->p, N);
  DALLOC(p->p2, N);
  DALLOC(p->ap, N);
  DALLOC(p->low, (size_t)v.Ho * v.Wo);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_kernel, 256, 0);
  int per_sm2 = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, power_kernel, 256, 0);
  p->coop_blocks = kSMs * std::max(1, std::min({per_sm, per_sm2, 2}));
  DALLOC(p->partial, (size_t)p->coop_blocks * 4);
  DALLOC(p->scal, 8);
  *out = p;
  return kOk;
}

int fepll_op_destroy(void* op) {
  OpPlan* p = static_cast<OpPlan*>(op);
  if (!p) return kOk;
  for (void* m : p->owned) cudaFree(m);
  delete p;
  return kOk;
}

// A^T y (operators.py:216-230); y: Ho x Wo, out: H x W
int fepll_op_adjoint(void* op, const double* y, double* out, void* stream) {
  OpPlan* p = static_cast<OpPlan*>(op);
  FEPLL_REQUIRE(p && y && out, "op_adjoint: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const OpView& v = p->v;
  const int64_t N = (int64_t)v.H * v.W;
  switch (v.kind) {
    case kIdentity:
    case kMask:
    case kGain:
      pixel_adjoint_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(y, v.pmap, out, N);
      FEPLL_LAUNCH();
      return kOk;
    case kConvolution:
      return fft_filter_2d(p, y, kFilterAdjoint, 0.0, out, nullptr, st);
    default:
      decimate_adjoint_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(v, y, out);
      FEPLL_LAUNCH();
      return kOk;
  }
}

// lambda = min(frob / (N l2sq), 250 sigma^2) with l2sq from the device power
// iteration started at v0 (operators.py:298-355); frob is the caller's
// closed form.  Synchronous (setup).
int fepll_op_lambda(void* op, const double* v0_host, double frob, double sigma, double* lam_out,
                    double* l2sq_out) {
  OpPlan* p = static_cast<OpPlan*>(op);
  FEPLL_REQUIRE(p && v0_host && lam_out, "op_lambda: bad arguments");
  FEPLL_REQUIRE(sigma > 0, "sigma must be positive");
  FEPLL_REQUIRE(frob != 0.0, "zero operator has no coupling parameter");
  const OpView& v = p->v;
  const int64_t N = (int64_t)v.H * v.W;
  FEPLL_CUDA(cudaMemcpy(p->r, v0_host, sizeof(double) * N, cudaMemcpyHostToDevice));
  PowerArgs a;
  a.nrm.o = v;
  a.nrm.shift = 0.0;
  a.nrm.lapc = 0.0;
  a.v = p->r;
  a.w = p->ap;
  a.low = p->low;
  a.partial = p->partial;
  a.out = p->scal;
  a.iters = 800;
  a.tol = 1e-9;
  int rc = coop_launch((const void*)power_kernel, &a, p, 0);
  if (rc) return rc;
  double l2 = 0.0;
  FEPLL_CUDA(cudaMemcpy(&l2, p->scal, sizeof(double), cudaMemcpyDeviceToHost));
  FEPLL_REQUIRE(l2 > 0.0, "operator spectral norm is zero");
  if (l2sq_out) *l2sq_out = l2;
  *lam_out = std::min(frob / ((double)N * l2), 250.0 * sigma * sigma);
  return kOk;
}

// init_estimate (operators.py:374-394): x = argmin ||Ax - y||^2 + c x^T L x,
// c = 0.2 sigma^2 / lam; FFT for identity/convolution, CG otherwise (x0 = A^T y).
int fepll_op_init(void* op, const double* y, const double* aty, double sigma, double lam,
                  double tol, int32_t maxit, double* x, double* info, void* stream) {
  OpPlan* p = static_cast<OpPlan*>(op);
  FEPLL_REQUIRE(p && y && aty && x, "op_init: bad arguments");
  FEPLL_REQUIRE(lam > 0, "lambda must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const OpView& v = p->v;
  const double c = 0.2 * sigma * sigma / lam;
  if (v.kind == kIdentity || v.kind == kConvolution) {
    FEPLL_REQUIRE(p->work != nullptr, "op_init: image too large for the FFT");
    return fft_filter_2d(p, y, kFilterInit, c, x, nullptr, st);
  }
  const int64_t N = (int64_t)v.H * v.W;
  FEPLL_CUDA(cudaMemcpyAsync(x, aty, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
  CgArgs a;
  a.nrm.o = v;
  a.nrm.shift = 0.0;
  a.nrm.lapc = c;
  a.rhs = aty;
  a.x = x;
  a.r = p->r;
  a.p = p->p;
  a.p2 = p->p2;
  a.ap = p->ap;
  a.low = p->low;
  a.partial = p->partial;
  a.out = info ? info : p->scal;
  a.status = nullptr;
  a.tol = tol;
  a.maxit = maxit;
  return coop_launch((const void*)cg_kernel, &a, p, st);
}

// solve_image_estimation for the non-pixel kinds (operators.py:288-295):
// convolution: x = ifft2(fft2(rhs) / (|khat|^2 + bs2)); decimate: CG on
// A^T A + bs2 I from x0 = x_tilde.  info (device, 4 doubles): iterations,
// residual, converged, finite.
int fepll_op_solve(void* op, const double* rhs, const double* xtilde, double bs2, double tol,
                   int32_t maxit, double* x, double* info, int32_t* status, void* stream) {
  OpPlan* p = static_cast<OpPlan*>(op);
  FEPLL_REQUIRE(p && rhs && x, "op_solve: bad arguments");
  FEPLL_REQUIRE(bs2 > 0, "beta_sigma2 must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const OpView& v = p->v;
  if (v.kind == kConvolution) return fft_filter_2d(p, rhs, kFilterSolve, bs2, x, status, st);
  FEPLL_REQUIRE(v.kind == kDecimate, "op_solve: pixel kinds are solved in fepll_aggregate");
  FEPLL_REQUIRE(xtilde != nullptr && info != nullptr, "op_solve: CG needs x_tilde and info");
  const int64_t N = (int64_t)v.H * v.W;
  FEPLL_CUDA(cudaMemcpyAsync(x, xtilde, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
  CgArgs a;
  a.nrm.o = v;
  a.nrm.shift = bs2;
  a.nrm.lapc = 0.0;
  a.rhs = rhs;
  a.x = x;
  a.r = p->r;
  a.p = p->p;
  a.p2 = p->p2;
  a.ap = p->ap;
  a.low = p->low;
  a.partial = p->partial;
  a.out = info;
  a.status = status;
  a.tol = tol;
  a.maxit = maxit;
  return coop_launch((const void*)cg_kernel, &a, p, st);
}

// diagnostics / tests: y = A^T A x + shift x
int fepll_op_normal(void* op, const double* xin, double shift, double* y, void* stream) {
  OpPlan* p = static_cast<OpPlan*>(op);
  FEPLL_REQUIRE(p && xin && y, "op_normal: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const OpView& v = p->v;
  const int64_t N = (int64_t)v.H * v.W;
  NormalArgs n;
  n.o = v;
  n.shift = shift;
  n.lapc = 0.0;
  normal_a_kernel<<<(unsigned)(((int64_t)v.Ho * v.Wo + 255) / 256), 256, 0, st>>>(n, xin, p->low);
  FEPLL_LAUNCH();
  normal_b_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(n, xin, p->low, y);
  FEPLL_LAUNCH();
  return kOk;
}

}  // extern "C"

