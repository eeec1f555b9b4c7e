// Kernel (d), staged form: reprojection of a batch through shared memory.
//
// Same result as aggregate_cover_kernel (aggregate.cu) — the per-pixel sum
// over the pixel's cover entries in ascending patch order, the lo == hi rule,
// the fused pixel update (patches.py:198-222, operators.py:281-287) — but the
// Zhat values are not gathered one 8-byte load per (pixel, entry).  A tile is
// one pixel row x `tw` columns; the rows of Zhat that cover it are `side`-
// element segments (window row dr of patch i = Zhat[i][dr*side ..]), each
// used by up to `side` neighbouring pixels.  Per image the CTA copies the
// tile's segments into a shared-memory stage with 16-byte cp.async (several
// images in flight), and each pixel then sums its entries out of the stage.
// The gather is latency-bound as one load per entry (ncu: long_scoreboard
// 55 %, 0.57 of HBM); staged, the loads are 16-byte, coalesced within a
// segment and NS-1 images deep.
//
// Plan-time tables (fepll_tiles_build, from the cover lists of
// aggregate.cu): per tile the sorted list of its segments (element offset
// i*P + dr*side inside an image's Zhat rows) and per cover entry the
// segment-local offset slot*side + dcol (uint16), i.e. the same entries
// re-addressed into the stage.  Every image of a batch shares the plan.
#include <algorithm>
#include <climits>

#include "common.cuh"

namespace fepll {

constexpr int kTileThreads = 256;   // = pixels per tile (tw)
constexpr int kTileRegEntries = 9;  // entries held in registers (more: loop over cover16)
constexpr int kTileMaxWords = 4096; // bitmap words of the build kernel (patch-id range 2^17)
constexpr int kTileStages = 4;

__device__ __forceinline__ void ta_cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void ta_cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void ta_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ta_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One CTA per tile: the tile's distinct patch ids (from its pixels' cover
// entries) get slots in ascending id order via a bitmap over [min id, max id]
// and a popcount scan; segment offsets and re-addressed entries follow.
__global__ void __launch_bounds__(kTileThreads)
tiles_build_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ entries, int P, int side,
                   int W, int tw, int n_chunks, int seg_cap, int32_t* __restrict__ seg_off,
                   int32_t* __restrict__ seg_cnt, uint16_t* __restrict__ cover16, int32_t* max_cnt,
                   int32_t* status) {
  __shared__ uint32_t bits[kTileMaxWords];
  __shared__ int32_t wscan[kTileMaxWords];
  __shared__ int red_mn[kTileThreads / 32], red_mx[kTileThreads / 32];
  __shared__ int s_mn, s_nw, s_total;
  const int tile = blockIdx.x;
  const int r = tile / n_chunks, j = tile - r * n_chunks;
  const int64_t p0 = (int64_t)r * W + (int64_t)j * tw;
  const int64_t p1 = min(p0 + tw, (int64_t)(r + 1) * W);
  const int e0 = ptr[p0], e1 = ptr[p1];
  int mn = INT_MAX, mx = -1;
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int id = entries[e] >> 8;
    mn = min(mn, id);
    mx = max(mx, id);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red_mn[threadIdx.x >> 5] = mn;
    red_mx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = INT_MAX, b = -1;
    for (int w = 0; w < kTileThreads / 32; ++w) {
      a = min(a, red_mn[w]);
      b = max(b, red_mx[w]);
    }
    s_mn = a;
    s_nw = b < a ? 0 : ((b - a) >> 5) + 1;
    if (s_nw > kTileMaxWords) {
      atomicOr(status, 8);  // patch-id range too wide for the bitmap: caller falls back
      s_nw = 0;
    }
  }
  __syncthreads();
  const int nw = s_nw, base = s_mn;
  if (nw == 0) {
    if (threadIdx.x == 0) seg_cnt[tile] = 0;
    return;
  }
  for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0u;
  __syncthreads();
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int d = (entries[e] >> 8) - base;
    atomicOr(&bits[d >> 5], 1u << (d & 31));
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // <= 4096 words, once per tile at plan time
    int acc = 0;
    for (int w = 0; w < nw; ++w) {
      wscan[w] = acc;
      acc += __popc(bits[w]);
    }
    s_total = acc;
  }
  __syncthreads();
  const int total = s_total;
  if (total > seg_cap) {
    if (threadIdx.x == 0) atomicOr(status, 8);
    return;
  }
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int v = entries[e];
    const int id = v >> 8, off = v & 255;
    const int d = id - base;
    const int slot = wscan[d >> 5] + __popc(bits[d >> 5] & ((1u << (d & 31)) - 1u));
    const int dr = off / side, dcol = off - dr * side;
    seg_off[(int64_t)tile * seg_cap + slot] = id * P + dr * side;  // same value from every entry of id
    cover16[e] = (uint16_t)(slot * side + dcol);
  }
  if (threadIdx.x == 0) {
    seg_cnt[tile] = total;
    atomicMax(max_cnt, total);
  }
}

// grid: (n_tiles, image groups); images [blockIdx.y*ipb, ...) of the batch.
// Stage slots rotate over NS; stage k holds image b0 + k (mod NS): the
// tile's segments (16-byte chunks, packed in slot order) and each pixel's
// A^T y / diagonal.  kDc: Zhat holds bare estimates (traces) and each
// segment's dc is staged next to it, added per value as aggregate.cu does.
// The per-image work is kept to the bare gather: chunk source offsets are
// resolved once per CTA (smem), entries are byte offsets into the stage.
template <typename ZT, bool kDc>
__global__ void __launch_bounds__(kTileThreads, 4)
aggregate_tiles_kernel(const ZT* __restrict__ Zhat, const double* __restrict__ dc, int n_local, int P,
                       const int32_t* __restrict__ ptr,
                       const uint16_t* __restrict__ cover16, const int32_t* __restrict__ seg_off,
                       const int32_t* __restrict__ seg_cnt, int seg_cap, int stage_elems, int stage_dc, int side,
                       int64_t zimg, int n_chunks, int batch, int H, int W, int r_begin,
                       const double* __restrict__ aty, const double* __restrict__ diag, double bs2,
                       int kind, double* __restrict__ x_out, double* __restrict__ xt_out,
                       int32_t* status, int ipb, int ns_alloc) {
  constexpr int kNS = kTileStages;
  constexpr int kVec = 16 / (int)sizeof(ZT);  // elements per 16-byte chunk
  extern __shared__ __align__(16) unsigned char ta_smem[];
  const int stage_bytes = stage_elems * (int)sizeof(ZT);
  const int dc_elems = kDc ? stage_dc : 0;  // doubles per stage (16-byte multiple)
  // ns_alloc = min(images per CTA, kNS) stages are allocated (the slots a
  // CTA's images cycle through)
  double* dcs = reinterpret_cast<double*>(ta_smem + (size_t)ns_alloc * stage_bytes);
  // per stage: this tile's A^T y (and diagonal) values, one per thread
  double* pxs = dcs + (size_t)ns_alloc * dc_elems;
  const int px_elems = diag ? 2 * kTileThreads : kTileThreads;
  uint32_t* coff = reinterpret_cast<uint32_t*>(pxs + (size_t)ns_alloc * px_elems);  // [n_chunk] byte offsets
  const int tile = blockIdx.x;
  const int rr = tile / n_chunks, j = tile - rr * n_chunks;
  const int c = j * kTileThreads + threadIdx.x;
  const bool valid = c < W;
  const int n_seg = seg_cnt[tile];
  const int cps = side / kVec;  // chunks per segment
  const int n_chunk = n_seg * cps;
  for (int q = threadIdx.x; q < n_chunk; q += kTileThreads) {
    const int sg = q / cps;
    coff[q] = (uint32_t)(seg_off[(int64_t)tile * seg_cap + sg] + (q - sg * cps) * kVec) * (uint32_t)sizeof(ZT);
  }
  const int64_t p = (int64_t)rr * W + c;
  int e0 = 0, cnt = 0;
  if (valid) {
    e0 = __ldg(ptr + p);
    cnt = __ldg(ptr + p + 1) - e0;
  }
  int off[kTileRegEntries];  // byte offsets into a stage
#pragma unroll
  for (int q = 0; q < kTileRegEntries; ++q)
    off[q] = (q < cnt) ? (int)__ldg(cover16 + e0 + q) * (int)sizeof(ZT) : 0;
  const bool pow2 = (cnt & (cnt - 1)) == 0;
  const double inv = cnt > 0 ? 1.0 / (double)cnt : 0.0;
  const int64_t pix0 = (int64_t)(r_begin + rr) * W + c;
  const int64_t img = (int64_t)H * W;
  const int b0 = blockIdx.y * ipb, b1 = min(batch, b0 + ipb);
  const double den = diag ? 0.0 : __dadd_rn(1.0, bs2);  // pixel-update denominator without a diagonal
  __syncthreads();  // coff
  auto issue = [&](int b, int slot) {
    const ZT* src = Zhat + (int64_t)b * zimg;
    const unsigned char* srcb = reinterpret_cast<const unsigned char*>(src);
    unsigned char* dst = ta_smem + (size_t)slot * stage_bytes;
    for (int q = threadIdx.x; q < n_chunk; q += kTileThreads) ta_cp_async16(dst + q * 16, srcb + coff[q]);
    if (kDc) {
      const double* dsrc = dc + (int64_t)b * n_local;
      double* ddst = dcs + (size_t)slot * dc_elems;
      for (int sg = threadIdx.x; sg < n_seg; sg += kTileThreads)
        ta_cp_async8(ddst + sg, dsrc + coff[sg * cps] / (uint32_t)(P * sizeof(ZT)));
    }
    if (valid) {
      double* pdst = pxs + (size_t)slot * px_elems + threadIdx.x;
      const int64_t pix = (int64_t)b * img + pix0;
      if (aty) ta_cp_async8(pdst, aty + pix);
      if (diag) ta_cp_async8(pdst + kTileThreads, diag + pix);
    }
  };
#pragma unroll
  for (int k = 0; k < kNS - 1; ++k) {
    if (b0 + k < b1) issue(b0 + k, k);
    ta_commit();
  }
  int slot = 0;
  for (int b = b0; b < b1; ++b) {
    ta_wait<kNS - 2>();
    __syncthreads();  // image b's stage complete; image b-1's slot free
    const int nb = b + kNS - 1;
    if (nb < b1) issue(nb, slot == 0 ? kNS - 1 : slot - 1);
    ta_commit();
    const unsigned char* sv = ta_smem + (size_t)slot * stage_bytes;
    const double* dv = dcs + (size_t)slot * dc_elems;
    const double* pv = pxs + (size_t)slot * px_elems + threadIdx.x;
    slot = slot == kNS - 1 ? 0 : slot + 1;
    if (!valid) continue;
    const double at = aty ? pv[0] : 0.0;
    auto val = [&](int o) {
      const double z = (double)*reinterpret_cast<const ZT*>(sv + o);
      return kDc ? __dadd_rn(z, dv[o / ((int)sizeof(ZT) * side)]) : z;
    };
    const int64_t pix = (int64_t)b * img + pix0;
    double xt;
    if (cnt == 0) {
      atomicOr(status, 1);
      xt = 0.0;
    } else {
      double v0, sum;
      bool ne = false;  // some entry differs from the first (lo != hi)
      if (cnt <= kTileRegEntries) {
        v0 = val(off[0]);
        sum = 0.0 + v0;
#pragma unroll
        for (int q = 1; q < kTileRegEntries; ++q) {
          if (q < cnt) {
            const double v = val(off[q]);
            sum += v;
            ne |= v != v0;
          }
        }
      } else {
        v0 = val(cover16[e0] * (int)sizeof(ZT));
        sum = 0.0 + v0;
        for (int q = 1; q < cnt; ++q) {
          const double v = val(cover16[e0 + q] * (int)sizeof(ZT));
          sum += v;
          ne |= v != v0;
        }
      }
      xt = !ne ? v0 : pow2 ? sum * inv : __ddiv_rn(sum, (double)cnt);
    }
    if (xt_out) xt_out[pix] = xt;
    const double rhs = __dadd_rn(at, __dmul_rn(bs2, xt));
    if (kind == 0) {
      const double x = __ddiv_rn(rhs, diag ? __dadd_rn(pv[kTileThreads], bs2) : den);
      if (!isfinite(x)) atomicOr(status, 2);
      if (x_out) x_out[pix] = x;
    } else if (x_out) {
      x_out[pix] = rhs;
    }
  }
  ta_wait<0>();
}

// dynamic shared memory of aggregate_tiles_kernel: NS stages of segments (+
// dc) and of the pixels' A^T y (+ diagonal), and the chunk offsets
static size_t tiles_smem_bytes(int max_seg, int side, int esize, bool with_dc, bool with_diag,
                               int ns = kTileStages) {
  const size_t seg_bytes = ((size_t)max_seg * side * esize + 15) / 16 * 16;
  return (size_t)ns * seg_bytes + (with_dc ? (size_t)ns * ((max_seg + 1) & ~1) * 8 : 0) +
         (size_t)ns * (with_diag ? 2 : 1) * kTileThreads * 8 + (size_t)max_seg * (side * esize / 16) * 4 + 16;
}

template <typename ZT>
static int aggregate_tiles_impl(const ZT* Zhat, const double* dc, int32_t n_local, const int32_t* ptr, const uint16_t* cover16,
                                const int32_t* seg_off, const int32_t* seg_cnt, int32_t seg_cap,
                                int32_t max_seg, int32_t P, int32_t side, int32_t zhat_rows,
                                int32_t batch, int32_t H, int32_t W, int32_t r_begin, int32_t r_end,
                                const double* aty, const double* diag, double bs2, int32_t kind,
                                double* x_out, double* xtilde_out, int32_t* status, void* stream) {
  FEPLL_REQUIRE(Zhat && ptr && cover16 && seg_off && seg_cnt && status, "aggregate_tiles: bad arguments");
  FEPLL_REQUIRE(kind == 0 || kind == 1, "aggregate_tiles: unknown kind");
  FEPLL_REQUIRE(0 <= r_begin && r_begin <= r_end && r_end <= H && batch >= 1, "aggregate_tiles: bad rows");
  FEPLL_REQUIRE(side >= 1 && side * side == P, "aggregate_tiles: P is not side^2");
  FEPLL_REQUIRE((side * sizeof(ZT)) % 16 == 0 && (reinterpret_cast<uintptr_t>(Zhat) & 15) == 0 &&
                    ((int64_t)zhat_rows * P * sizeof(ZT)) % 16 == 0,
                "aggregate_tiles: Zhat segments are not 16-byte aligned (use fepll_aggregate_cover)");
  FEPLL_REQUIRE(max_seg >= 0 && max_seg <= seg_cap, "aggregate_tiles: bad segment count");
  if (r_end == r_begin) return kOk;
  const int n_chunks = (W + kTileThreads - 1) / kTileThreads;
  const int64_t n_tiles = (int64_t)(r_end - r_begin) * n_chunks;
  FEPLL_REQUIRE(n_tiles < (int64_t(1) << 31), "aggregate_tiles: too many tiles");
  const int stage_elems = ((max_seg * side * (int)sizeof(ZT) + 15) / 16) * 16 / (int)sizeof(ZT);
  const int stage_dc = (max_seg + 1) & ~1;
  // image groups: enough CTAs to fill the GPU, at least 8 images per group
  // (a single image: one CTA per tile, the latency hidden by resident CTAs)
  int groups = 1;
  while (n_tiles * groups < 4 * kSMs * 4 && batch / (groups * 2) >= 8) groups *= 2;
  const int ipb = (batch + groups - 1) / groups;
  const int ns_alloc = std::min(ipb, kTileStages);
  const size_t smem = tiles_smem_bytes(max_seg, side, (int)sizeof(ZT), dc != nullptr, diag != nullptr, ns_alloc);
  FEPLL_REQUIRE(smem <= 227 * 1024, "aggregate_tiles: tile segments exceed shared memory");
  auto k = dc ? aggregate_tiles_kernel<ZT, true> : aggregate_tiles_kernel<ZT, false>;
  static bool attr_set[2] = {false, false};  // per instantiation; set before any graph capture
  if (!attr_set[dc ? 1 : 0]) {
    FEPLL_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set[dc ? 1 : 0] = true;
  }
  dim3 grid((unsigned)n_tiles, (unsigned)((batch + ipb - 1) / ipb));
  k<<<grid, kTileThreads, smem, (cudaStream_t)stream>>>(
      Zhat, dc, n_local, P, ptr, cover16, seg_off, seg_cnt, seg_cap, stage_elems, stage_dc, side, (int64_t)zhat_rows * P, n_chunks,
      batch, H, W, r_begin, aty, diag, bs2, kind, x_out, xtilde_out, status, ipb, ns_alloc);
  FEPLL_LAUNCH();
  return kOk;
}

}  // namespace fepll

extern "C" int32_t fepll_tiles_seg_cap(int32_t side, int32_t spacing, int32_t half) {
  using namespace fepll;
  // candidate nominal rows of one pixel row (+ the clamped last row) x
  // candidate columns of a tw-pixel run (+ the last column)
  const int rows = (side + 2 * half + spacing - 1) / spacing + 2;
  const int cols = (kTileThreads + side + 2 * half + spacing - 1) / spacing + 2;
  return rows * cols;
}

extern "C" int32_t fepll_tiles_width(void) { return fepll::kTileThreads; }

extern "C" int64_t fepll_tiles_smem_bytes(int32_t max_seg, int32_t side, int32_t elem_bytes, int32_t with_dc,
                                          int32_t with_diag) {
  return (int64_t)fepll::tiles_smem_bytes(max_seg, side, elem_bytes, with_dc != 0, with_diag != 0);
}

extern "C" int fepll_tiles_build(const int32_t* ptr, const int32_t* entries, int32_t P, int32_t side,
                                 int32_t W, int32_t rows, int32_t seg_cap, int32_t* seg_off,
                                 int32_t* seg_cnt, uint16_t* cover16, int32_t* max_cnt,
                                 int32_t* status, void* stream) {
  using namespace fepll;
  FEPLL_REQUIRE(ptr && entries && seg_off && seg_cnt && cover16 && max_cnt && status,
                "tiles_build: bad arguments");
  FEPLL_REQUIRE(side >= 1 && side * side == P && P <= 256 && W >= 1 && rows >= 0 && seg_cap >= 1,
                "tiles_build: bad geometry");
  FEPLL_REQUIRE((int64_t)seg_cap * side <= 65536, "tiles_build: segment slots exceed 16-bit offsets");
  if (rows == 0) return kOk;
  const int n_chunks = (W + kTileThreads - 1) / kTileThreads;
  const int64_t n_tiles = (int64_t)rows * n_chunks;
  FEPLL_REQUIRE(n_tiles < (int64_t(1) << 31), "tiles_build: too many tiles");
  cudaStream_t st = (cudaStream_t)stream;
  FEPLL_CUDA(cudaMemsetAsync(max_cnt, 0, sizeof(int32_t), st));
  tiles_build_kernel<<<(unsigned)n_tiles, kTileThreads, 0, st>>>(ptr, entries, P, side, W, kTileThreads,
                                                                  n_chunks, seg_cap, seg_off, seg_cnt,
                                                                  cover16, max_cnt, status);
  FEPLL_LAUNCH();
  return kOk;
}

extern "C" int fepll_aggregate_tiles(const double* Zhat, const float* Zhat32, const double* dc,
                                     int32_t n_local, const int32_t* ptr,
                                     const uint16_t* cover16, const int32_t* seg_off,
                                     const int32_t* seg_cnt, int32_t seg_cap, int32_t max_seg, int32_t P,
                                     int32_t zhat_rows, int32_t batch, int32_t H, int32_t W,
                                     int32_t r_begin, int32_t r_end, const double* aty, const double* diag,
                                     double bs2, int32_t kind, double* x_out, double* xtilde_out,
                                     int32_t* status, void* stream) {
  FEPLL_REQUIRE((Zhat == nullptr) != (Zhat32 == nullptr), "aggregate_tiles: exactly one of Zhat / Zhat32");
  int side = 1;
  while (side * side < P) ++side;
  if (Zhat32)
    return fepll::aggregate_tiles_impl(Zhat32, dc, n_local, ptr, cover16, seg_off, seg_cnt, seg_cap, max_seg, P, side,
                                       zhat_rows, batch, H, W, r_begin, r_end, aty, diag, bs2, kind, x_out,
                                       xtilde_out, status, stream);
  return fepll::aggregate_tiles_impl(Zhat, dc, n_local, ptr, cover16, seg_off, seg_cnt, seg_cap, max_seg, P, side,
                                     zhat_rows, batch, H, W, r_begin, r_end, aty, diag, bs2, kind, x_out,
                                     xtilde_out, status, stream);
}
