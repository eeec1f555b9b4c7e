// FP64 mixed-radix Stockham FFT, one CTA per 1-D transform in shared memory.
//
// Replaces numpy's pocketfft calls of the reference operators
// (pkg/src/fepll/operators.py:91-100, 196-197, 288-292, 336, 383-389).
// A length-N transform is factored into radices 4, 2, 3, 5, 7 and any
// remaining primes; each stage reads with stride N/R, applies the stage
// twiddles, does an R-point DFT and writes the autosorted output
//   d1[(j/Ns)*Ns*R + j%Ns + r*Ns] = DFT_R(tw .* d0[j + r*N/R])
// (Stockham, decimation in time).  Twiddles and roots are FP64 tables built
// on the host with libm cos/sin.
#pragma once
#include <vector>

#include "common.cuh"

namespace fepll {

constexpr int kFftMaxN = 4096;
constexpr int kFftMaxStages = 24;
constexpr int kFftMaxRadix = 64;

struct FftDim {
  int n = 0;
  int stages = 0;
  int radix[kFftMaxStages];
  int ns[kFftMaxStages];
  int tw_off[kFftMaxStages];   // complex offsets into the twiddle table
  int root_off[kFftMaxStages]; // complex offsets into the root table
  const double2* tw = nullptr;
  const double2* root = nullptr;
};

// host: factor n and build the tables (uploaded into owned device memory)
int fft_dim_build(int n, FftDim* out, std::vector<void*>* owned);

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// in-place forward transform of d0 (length fd.n) using d1 as scratch; the
// result ends in the returned buffer.  All threads of the CTA participate.
__device__ inline double2* fft_smem(const FftDim& fd, double2* d0, double2* d1) {
  const int N = fd.n;
  for (int s = 0; s < fd.stages; ++s) {
    const int R = fd.radix[s];
    const int Ns = fd.ns[s];
    const int M = N / R;
    const double2* tw = fd.tw + fd.tw_off[s];
    const double2* root = fd.root + fd.root_off[s];
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      const int jj = j % Ns;
      const int idx = (j / Ns) * Ns * R + jj;
      if (R == 2) {
        double2 a = d0[j], b = cmul(d0[j + M], tw[jj * 2 + 1]);
        d1[idx] = make_double2(a.x + b.x, a.y + b.y);
        d1[idx + Ns] = make_double2(a.x - b.x, a.y - b.y);
      } else if (R == 4) {
        double2 v0 = d0[j];
        double2 v1 = cmul(d0[j + M], tw[jj * 4 + 1]);
        double2 v2 = cmul(d0[j + 2 * M], tw[jj * 4 + 2]);
        double2 v3 = cmul(d0[j + 3 * M], tw[jj * 4 + 3]);
        const double2 s02 = make_double2(v0.x + v2.x, v0.y + v2.y);
        const double2 d02 = make_double2(v0.x - v2.x, v0.y - v2.y);
        const double2 s13 = make_double2(v1.x + v3.x, v1.y + v3.y);
        const double2 d13 = make_double2(v1.x - v3.x, v1.y - v3.y);
        // forward: X1 = d02 - i d13, X3 = d02 + i d13
        d1[idx] = make_double2(s02.x + s13.x, s02.y + s13.y);
        d1[idx + Ns] = make_double2(d02.x + d13.y, d02.y - d13.x);
        d1[idx + 2 * Ns] = make_double2(s02.x - s13.x, s02.y - s13.y);
        d1[idx + 3 * Ns] = make_double2(d02.x - d13.y, d02.y + d13.x);
      } else {
        double2 v[kFftMaxRadix];
        for (int r = 0; r < R; ++r) {
          const double2 x = d0[j + r * M];
          v[r] = r ? cmul(x, tw[jj * R + r]) : x;
        }
        for (int k = 0; k < R; ++k) {
          double2 acc = v[0];
          int e = 0;
          for (int r = 1; r < R; ++r) {
            e += k;
            if (e >= R) e -= R;
            const double2 w = root[e];
            acc.x += v[r].x * w.x - v[r].y * w.y;
            acc.y += v[r].x * w.y + v[r].y * w.x;
          }
          d1[idx + k * Ns] = acc;
        }
      }
    }
    __syncthreads();
    double2* tmp = d0;
    d0 = d1;
    d1 = tmp;
  }
  return d0;
}

}  // namespace fepll
