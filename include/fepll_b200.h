/*
 * fepll_b200.h — C ABI of the B200-native FEPLL restoration loop.
 *
 * Every entry point takes plain pointers, sizes and a cudaStream_t (passed
 * as void*); device pointers are caller-owned (the Python host passes
 * torch tensor data pointers).  Return codes: 0 ok, 3 data error,
 * 4 numerical error, 5 CUDA error; fepll_last_error() returns the message
 * of the last failure on the calling thread.
 *
 * Each entry point replaces one function of the reference hot path
 * (/root/reference/pkg/src/fepll/...), cited beside its declaration.
 */
#ifndef FEPLL_B200_H
#define FEPLL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fepll_plan_s* fepll_plan_t;

/* Packed tree + model, built on the host from GmmTree/GmmModel
 * (tree.py:253-276 BFS order, gmm.py:96-155 component fields).
 * Group g of an internal node u = its children's kept bases concatenated
 * (child order), stored P x width row-major at grp_off64[u] in grp_basis. */
typedef struct fepll_plan_desc {
  int32_t patch_dim;        /* P */
  int32_t n_nodes;          /* BFS nodes of the tree */
  int32_t n_components;     /* K (model components == tree leaves) */
  int32_t iterations;       /* T: beta schedule length */
  const int32_t* child_start;   /* [n_nodes] */
  const int32_t* child_count;   /* [n_nodes] */
  const int32_t* child_list;    /* [n_nodes-1] BFS ids */
  const int32_t* leaf_index;    /* [n_nodes] -1 internal */
  const int32_t* depth;         /* [n_nodes] */
  const int32_t* node_rank;     /* [n_nodes] */
  const int32_t* grp_width;     /* [n_nodes] sum of child ranks (0 for leaves) */
  const int32_t* grp_col_off;   /* [n_nodes] group column offset */
  const int32_t* child_col_off; /* [n_nodes] column offset inside the parent's group */
  const int64_t* grp_off64;     /* [n_nodes] element offset of the group block */
  const double* grp_basis;      /* [sum P*width] */
  int64_t grp_basis_len;
  int32_t grp_cols_total;
  const double* node_const;     /* [T][n_nodes] gmm.py:304-306 */
  const double* node_nu_tail;   /* [T][n_nodes] gmm.py:293 */
  const double* grp_sqw;        /* [T][grp_cols_total] gmm.py:303 */
  const int32_t* model_rank;    /* [K] */
  const int32_t* model_col_off; /* [K] */
  const int64_t* model_off64;   /* [K] element offset of P x r_k block */
  const double* model_basis;    /* [sum P*r_k] */
  int64_t model_basis_len;
  int32_t model_cols_total;
  const double* model_shrink;   /* [T][model_cols_total] gmm.py:307 */
  const double* model_gamma_tail; /* [T][K] gmm.py:297 */
  const float* grp_tc_hi;       /* tcgen05 operand images (may be NULL) */
  const float* grp_tc_lo;
  int64_t grp_tc_len;
  const int64_t* grp_tc_off;    /* [n_nodes] float offset of the node's B image */
  const int32_t* grp_tc_npad;   /* [n_nodes] padded width (multiple of 16) */
  const int32_t* grp_tc_child_col; /* [n_nodes] 16-aligned column of a child in its parent's image */
  const float* grp_tc_w;        /* [T][grp_tc_w_cols] FP32 column weights (0 on padding) */
  const int32_t* grp_tc_w_off;  /* [n_nodes] first weight column of a node's image */
  int32_t grp_tc_w_cols;
  /* bf16 [lo | hi] images of the mixed-precision scorer, same layout and
   * length as grp_tc_hi (may be NULL: the level kernel then uses 3xTF32) */
  const float* grp_tc_x;
} fepll_plan_desc;

int fepll_abi_version(void);
/* number of kernels this library has launched in the process (bench evidence) */
int64_t fepll_launch_count(void);
const char* fepll_last_error(void);

/* tree.py:387-434 + gmm.py:275-307: owns packed bases and per-beta constants. */
int fepll_plan_create(const fepll_plan_desc* desc, fepll_plan_t* out);
/* scratch for up to max_patches patches per select call */
int fepll_plan_reserve(fepll_plan_t plan, int64_t max_patches);
int fepll_plan_destroy(fepll_plan_t plan);
/* Per-plan kernel choices (no process-global state): A/B switches between
 * kernel variants that produce bitwise-identical results, plus the Wiener
 * output form.  Names and values:
 *   select_variant 0 | 1 | 2  tree-level kernel: select_ws.cu (3xTF32),
 *                             select_ws2.cu (tf32 + bf16 cross pass, default 1),
 *                             ws2 on levels of <= 16 nodes and ws elsewhere;
 *   seg_sq 0 | 1              ws2 levels pass ||z||^2 in segment order (default 1);
 *   wiener_pair 0 | 1         two 64-row Wiener CTAs per SM when they fit (1);
 *   wiener_rw 8 | 16          rows per warp in that configuration (8);
 *   wiener_split 0 | 1        Wiener warp pairs share 16 rows and issue m16n8k8
 *                             DMMAs, C crossing through shared memory (1), or
 *                             8-row warps with m8n8k4 (0, default: measured
 *                             2 % faster) — bitwise the same;
 *   wiener_tc 0 | 1           fepll_wiener_f32 runs on tcgen05 with 3xTF32 products
 *                             (wiener_tc.cu; P % 16 == 0, P <= 64, ranks <= 64)
 *                             instead of the FP64 DMMA kernel — NOT bitwise the
 *                             same: ~1e-6 relative on the estimates;
 *   wiener_ws 0 | 1 | 2       FP64 Wiener (P = 64): warp-specialised kernel — 12 compute
 *                             warps + 2 loader warps, one CTA per SM, no CTA barrier
 *                             between tiles — bitwise the two-CTA kernel; 2 (default):
 *                             from 2^20 patches per call (measured +3 % there, -8 %
 *                             at 8 x 1024^2);
 *   wiener_xw 0 | 1           Wiener reads 8x8 windows of x instead of Z64 (0);
 *   wiener_add_dc 0 | 1       fepll_wiener writes est + dc (1) or the bare
 *                             estimates (0: the trace's `estimates`; pass dc
 *                             to the aggregation then);
 *   l2_prefetch 0 | 1 | 2     ws2 tree-level loaders prefetch each tile's rows
 *                             into L2 three tiles before copying them, per
 *                             line (1) or one bulk prefetch per row (2);
 *                             measured slower, default 0;
 *   aggregate_variant 0|1|2   batch reprojection kernel the host uses:
 *                             fepll_aggregate_cover_ex (0: one thread per pixel
 *                             over the images, 1: one per (pixel, image)) or
 *                             fepll_aggregate_tiles (2: staged in shared memory,
 *                             default; batches only);
 *   pdl 0 | 1                 tree-level and re-scoring kernels launched with
 *                             programmatic dependent launch: each one's prologue
 *                             overlaps its predecessor's tail (default 1);
 *   defer 0 | 1               (ws2 / select_tc trees, select_variant 1)
 *                             uncertified decisions are routed by the
 *                             tensor-core argmin and verified in FP64 after the
 *                             last level, mis-routed patches re-descended (1,
 *                             default), or re-scored after every level (0) —
 *                             the same labels, buckets and counts;
 *   defer_test 0 | 1          test hook: the uncertified rows are routed
 *                             provisionally to a wrong child, so the
 *                             verification has to repair each of them (0);
 *   rescore_by_node 0 | 1     FP64 re-scoring grouped by tree node, the node's
 *                             group matrix staged in shared memory (measured
 *                             slower, default 0).
 * Unknown names or out-of-range values: data error. */
int fepll_plan_set_option(fepll_plan_t plan, const char* name, int64_t value);
int fepll_plan_get_option(fepll_plan_t plan, const char* name, int64_t* value);
/* Timing of the tree-level kernels (kernel (b)): with capacity > 0 the next
 * `capacity` level launches of fepll_select are bracketed by CUDA events on
 * the caller's stream; _read returns their summed duration and count and
 * resets.  capacity 0 turns it off. */
int fepll_plan_profile(fepll_plan_t plan, int32_t capacity);
int fepll_plan_profile_read(fepll_plan_t plan, double* total_ms, int32_t* launches);

/* patches.py:89-132: the sampling plan of iteration t on the device,
 * bit-identical to jittered_grid(H, W, side^2, spacing,
 * Generator(Philox(key=[seed, t]))) (jittered != 0) or regular_grid.
 * key0/key1: the Philox key words numpy derives from [seed, t].
 * anchors: [n_rows*n_cols][2] int32 (row, col), nominal row-major order.
 * scratch: device int32[fepll_grid_scratch_ints()].  status bit 4 is set if
 * more draws were rejected than the fix-up list holds (never expected).
 * threshold_override: 0, or a Lemire rejection threshold used instead of
 * (2^32 - n) mod n (test hook exercising the rejection fix-up). */
int fepll_grid_scratch_ints(void);
int fepll_sample_grid(uint64_t key0, uint64_t key1, int32_t H, int32_t W, int32_t side,
                      int32_t spacing, int32_t jittered, uint32_t threshold_override,
                      int32_t* anchors, int32_t* scratch, int32_t* status, void* stream);

/* patches.py:167-183 (extract + _row_mean pairwise fold):
 * x: [batch][H][W] fp64; anchors: [n][2] int32 (row, col);
 * grid_cols: unused (kept for ABI stability), pass 0;
 * outputs (any may be NULL): Z64 [batch*n][P], Z32 [batch*n][z32_pitch]
 * (zero-padded past P; the tcgen05 scorer reads 128-byte K atoms), dc, sq.
 * Any pitch >= P and any element alignment are accepted; the fast kernel
 * (paired 16-/8-byte row stores) runs when Z64 is 16-byte aligned, Z32
 * 8-byte aligned and z32_pitch even, a per-row-store kernel otherwise. */
int fepll_extract(const double* x, int32_t batch, int32_t H, int32_t W, int32_t side,
                  const int32_t* anchors, int32_t n, int32_t grid_cols, double* Z64, float* Z32,
                  int32_t z32_pitch, double* dc, double* sq, void* stream);

/* tree.py:387-434 (greedy descent, first-min tie break) over n_total =
 * batch * n_img patches whose values are re-extracted from the FP64 images x
 * ([batch][H][W]) at anchors ([n_img][2]) minus dc (patches.py:178).
 * mode 0: exact FP64 scoring; mode 1: tcgen05 tensor-core scoring (P <= 64:
 * one kind::tf32 pass + one bf16 cross pass, select_ws2.cu; P <= 128:
 * 3xTF32) with a certified argmin and FP64 re-scoring of every decision the
 * certificate does not cover (needs Z32, the FP32 patch rows written by
 * fepll_extract).  Z64 (optional, the FP64 rows of fepll_extract, bitwise
 * the re-extracted values) saves the exact / re-scoring paths the window
 * reads.  guard <= 0 selects the default bound 2^-16 (tc_epi.cuh).
 * labels: [n_total] int32 leaf indices.  leaf_counts (optional, device
 * int64 [K]) receives the label histogram. */
int fepll_select(fepll_plan_t plan, int32_t t, const double* x, int32_t H, int32_t W,
                 const int32_t* anchors, int32_t n_img, const double* dc, const double* sq,
                 const float* Z32, const double* Z64, int64_t n_total, int32_t mode, double guard,
                 int32_t* labels, int64_t* leaf_counts, void* stream);

/* diagnostics: per-level count of decisions the last tensor-mode select sent
 * to exact FP64 re-scoring (dst[0..61]), the patches the deferred
 * verification re-descended (dst[62]) and its overflow flags (dst[63]);
 * dst: device int32[64]. */
int fepll_select_rescored(fepll_plan_t plan, int32_t* dst, void* stream);

/* gmm.py:352-359 / solver.py:233-241: FP64 Wiener estimates of the patches
 * under their labels, grouped by label (the leaf buckets of the last select).
 * With Z64 (the FP64 patch rows of fepll_extract) it runs on the FP64 tensor
 * cores (DMMA); without, on the DMMA kernel reading the windows of x when
 * fepll_wiener_reads_image(plan), else on CUDA cores re-extracting from x.  Zhat receives
 * est + dc (patches.py:198-222's reprojection values), ready for
 * fepll_aggregate* with dc == NULL.  Zhat holds zhat_rows (>= n_img) rows of
 * P doubles per image: patch b*n_img + i is row b*zhat_rows + i (a padded
 * image pitch keeps the images' rows off power-of-two strides). */
/* 1 when fepll_wiener, given Z64 == NULL, runs the DMMA kernel on 8 x 8
 * windows of x (minus dc) itself — P = 64 — so fepll_extract need not write
 * the FP64 rows; 0 when it needs Z64 for the DMMA path. */
int fepll_wiener_reads_image(fepll_plan_t plan);

int fepll_wiener(fepll_plan_t plan, int32_t t, const double* x, int32_t H, int32_t W,
                 const int32_t* anchors, int32_t n_img, const double* dc, const double* Z64,
                 int64_t n_total, double* Zhat, int32_t zhat_rows, void* stream);

/* FP32-state mode (opt-in, Restorer(precision="fp32-state")): the Wiener
 * kernel reads the FP32 patch rows of fepll_extract (z32_pitch floats per
 * row, 16-byte aligned) and writes est + dc rounded once to FP32; the
 * arithmetic in between is the FP64 DMMA of fepll_wiener, or — plan option
 * wiener_tc — three kind::tf32 tcgen05 passes per product with FP32
 * accumulation (HBM-bound instead of FP64-pipe-bound). */
int fepll_wiener_f32(fepll_plan_t plan, int32_t t, const double* x, int32_t H, int32_t W,
                     const int32_t* anchors, int32_t n_img, const double* dc, const float* Z32,
                     int32_t z32_pitch, int64_t n_total, float* Zhat, int32_t zhat_rows, void* stream);

/* patches.py:198-222 (+ operators.py:284-287 when kind==0):
 * per-pixel ordered gather of (Zhat + dc) over covering anchors; dc may be
 * NULL when Zhat already holds est + dc (fepll_wiener's output).
 * grid geometry: n_rows x n_cols nominal anchors, spacing, half, side.
 * kind 0: x = (aty + bs2*xt) / (diag + bs2)  (pixel-diagonal update fused)
 * kind 1: rhs = aty + bs2*xt (FFT/CG kinds).  Outputs may be NULL. */
int fepll_aggregate(const double* Zhat, const double* dc, const int32_t* anchors,
                    int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                    int32_t side, int32_t batch, int32_t H, int32_t W,
                    const double* aty, const double* diag, double bs2, int32_t kind,
                    double* x_out, double* xtilde_out, int32_t* status, void* stream);

/* Strip form of fepll_aggregate (one image split by pixel rows across
 * ranks): the local image ([batch][H][W]) is global rows [row0, row0+H) of an
 * image with H_glob rows; Zhat/dc/anchors hold the patches of global nominal
 * anchor rows [a_first, a_first + n_local_rows) (anchor rows local to the
 * strip); n_rows is the global nominal row count.  Only local rows
 * [r_begin, r_end) are written, each bit-identical to the unsplit result. */
int fepll_aggregate_strip(const double* Zhat, const double* dc, const int32_t* anchors,
                          int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                          int32_t side, int32_t batch, int32_t H, int32_t W,
                          int32_t row0, int32_t H_glob, int32_t a_first,
                          int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                          const double* aty, const double* diag, double bs2, int32_t kind,
                          double* x_out, double* xtilde_out, int32_t* status, void* stream);

/* FP32-state form: Zhat holds FP32 est + dc; sums run in FP64 as above. */
int fepll_aggregate_strip_f32(const float* Zhat, const double* dc, const int32_t* anchors,
                              int32_t n_rows, int32_t n_cols, int32_t spacing, int32_t half,
                              int32_t side, int32_t batch, int32_t H, int32_t W,
                              int32_t row0, int32_t H_glob, int32_t a_first,
                              int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                              const double* aty, const double* diag, double bs2, int32_t kind,
                              double* x_out, double* xtilde_out, int32_t* status, void* stream);

/* Cover lists (CSR) of a sampling plan: for local rows [r_begin, r_end) of a
 * (strip of an) image, the anchors covering each pixel in ascending patch
 * order (the np.bincount order of patches.py:213-220), entry = local patch
 * index << 8 | (dr*side + dcol).  The plan is shared by all images of a
 * batch, so this is built once per iteration's grid.  ptr: [npx + 1],
 * entries: >= n_local_rows*n_cols*side^2, scratch: int32
 * [fepll_cover_scratch_ints(npx)], npx = (r_end - r_begin) * W.
 * Geometry arguments as fepll_aggregate_strip. */
int64_t fepll_cover_scratch_ints(int64_t n_pixels);
int fepll_cover_build(const int32_t* anchors, int32_t n_rows, int32_t n_cols, int32_t spacing,
                      int32_t half, int32_t side, int32_t W, int32_t row0, int32_t H_glob,
                      int32_t a_first, int32_t n_local_rows, int32_t r_begin, int32_t r_end,
                      int32_t* ptr, int32_t* entries, int64_t entries_cap, int32_t* scratch,
                      void* stream);

/* fepll_aggregate over cover lists (bit-identical results): Zhat holds
 * zhat_rows (>= n_local) rows per image of which the first n_local are the
 * image's patches, dc n_local per image; images [batch][H][W]; rows
 * [r_begin, r_end). */
int fepll_aggregate_cover(const double* Zhat, const double* dc, const int32_t* ptr,
                          const int32_t* entries, int32_t P, int32_t n_local, int32_t zhat_rows,
                          int32_t batch,
                          int32_t H, int32_t W, int32_t r_begin, int32_t r_end,
                          const double* aty, const double* diag, double bs2, int32_t kind,
                          double* x_out, double* xtilde_out, int32_t* status, void* stream);

/* fepll_aggregate_cover with the Zhat element type and batch kernel
 * explicit: exactly one of Zhat (FP64) / Zhat32 (FP32) non-NULL; variant 0:
 * one thread per pixel looping over the images, 1: one thread per (pixel,
 * image).  Bitwise-identical results. */
int fepll_aggregate_cover_ex(const double* Zhat, const float* Zhat32, const double* dc,
                             const int32_t* ptr, const int32_t* entries, int32_t P, int32_t n_local,
                             int32_t zhat_rows, int32_t batch, int32_t H, int32_t W, int32_t r_begin,
                             int32_t r_end, const double* aty, const double* diag, double bs2,
                             int32_t kind, double* x_out, double* xtilde_out, int32_t* status,
                             int32_t variant, void* stream);

/* Staged reprojection of a batch (kernel (d), csrc/aggregate_tiles.cu):
 * the same results as fepll_aggregate_cover_ex, read through shared memory.
 * A tile is one pixel row x fepll_tiles_width() columns; fepll_tiles_build
 * turns a plan's cover lists (ptr, entries over `rows` = r_end - r_begin
 * rows) into per-tile segment tables — seg_off [n_tiles][seg_cap] (element
 * offset patch*P + dr*side of a window row inside an image's Zhat rows),
 * seg_cnt [n_tiles], cover16 [entries] (the entry re-addressed into the
 * tile's stage) — and writes the largest count to *max_cnt (device int).
 * seg_cap >= fepll_tiles_seg_cap(side, spacing, half); status bit 8: a tile
 * does not fit the tables (use fepll_aggregate_cover_ex for that plan).
 * n_tiles = rows * ceil(W / fepll_tiles_width()).  fepll_aggregate_tiles
 * needs 16-byte aligned window rows (side * sizeof(element) % 16 == 0);
 * exactly one of Zhat / Zhat32; dc (n_local per image) or NULL as in
 * fepll_aggregate_cover. */
int32_t fepll_tiles_width(void);
int32_t fepll_tiles_seg_cap(int32_t side, int32_t spacing, int32_t half);
/* dynamic shared memory fepll_aggregate_tiles needs for a plan (must stay
 * <= 227 KB; larger plans keep fepll_aggregate_cover_ex) */
int64_t fepll_tiles_smem_bytes(int32_t max_seg, int32_t side, int32_t elem_bytes, int32_t with_dc,
                               int32_t with_diag);
int fepll_tiles_build(const int32_t* ptr, const int32_t* entries, int32_t P, int32_t side, int32_t W,
                      int32_t rows, int32_t seg_cap, int32_t* seg_off, int32_t* seg_cnt,
                      uint16_t* cover16, int32_t* max_cnt, int32_t* status, void* stream);
int fepll_aggregate_tiles(const double* Zhat, const float* Zhat32, const double* dc, int32_t n_local,
                          const int32_t* ptr, const uint16_t* cover16, const int32_t* seg_off,
                          const int32_t* seg_cnt, int32_t seg_cap, int32_t max_seg, int32_t P,
                          int32_t zhat_rows, int32_t batch, int32_t H, int32_t W, int32_t r_begin,
                          int32_t r_end, const double* aty, const double* diag, double bs2,
                          int32_t kind, double* x_out, double* xtilde_out, int32_t* status,
                          void* stream);

/* FP32-state form of fepll_aggregate_cover (FP32 Zhat, FP64 sums). */
int fepll_aggregate_cover_f32(const float* Zhat, const double* dc, const int32_t* ptr,
                              const int32_t* entries, int32_t P, int32_t n_local, int32_t zhat_rows,
                              int32_t batch, int32_t H, int32_t W, int32_t r_begin, int32_t r_end,
                              const double* aty, const double* diag, double bs2, int32_t kind,
                              double* x_out, double* xtilde_out, int32_t* status, void* stream);

/* ---- degradation operators (operators.py:51-394); handle = opaque plan.
 * kind: 0 identity, 1 convolution, 2 mask, 3 gain, 4 decimate (factor).
 * taps: [kh][kw] host kernel (kinds 1, 4); pixel_map: [H][W] host (2, 3). */
int fepll_op_create(int32_t kind, int32_t H, int32_t W, int32_t factor, const double* taps,
                    int32_t kh, int32_t kw, const double* pixel_map, void** out);
int fepll_op_destroy(void* op);
/* apply_adjoint (operators.py:216-230): y [Ho][Wo] -> out [H][W] (device) */
int fepll_op_adjoint(void* op, const double* y, double* out, void* stream);
/* lambda_param (operators.py:342-355): power iteration from the host start
 * vector v0 [H][W] on the device; frob = ||A^T A||_F^2 (closed form).
 * Synchronous; writes lambda and the power-iteration estimate l2sq. */
int fepll_op_lambda(void* op, const double* v0_host, double frob, double sigma, double* lam_out,
                    double* l2sq_out);
/* init_estimate (operators.py:374-394); info: device double[4]
 * (iterations, residual, converged, finite) for the CG kinds. */
int fepll_op_init(void* op, const double* y, const double* aty, double sigma, double lam,
                  double tol, int32_t maxit, double* x, double* info, void* stream);
/* solve_image_estimation for convolution (FFT) and decimate (CG from
 * x0 = x_tilde) (operators.py:273-295); rhs = A^T y + bs2 x_tilde. */
int fepll_op_solve(void* op, const double* rhs, const double* xtilde, double bs2, double tol,
                   int32_t maxit, double* x, double* info, int32_t* status, void* stream);
/* normal_apply (operators.py:233-235) + shift: y = A^T A x + shift x */
int fepll_op_normal(void* op, const double* x, double shift, double* y, void* stream);

/* ---- offline search-tree construction (tree.py:99-200, build_tree's
 * device parts; csrc/tree_build.cu).
 * fepll_tree_kl: inv, cov: device [K][P*P] FP64 (the dense inverses and
 * covariances of tree.py:72-87); t_scratch: device [K][K]; kl: device
 * [K][K] = 0.5 (t + t^T) - P, zero diagonal, t[a][b] = Tr(C_a^-1 C_b)
 * (pairwise_symmetric_kl, tree.py:99-107). */
int fepll_tree_kl(const double* inv, const double* cov, int32_t K, int32_t P, double* t_scratch,
                  double* kl, void* stream);
/* fepll_cluster_swap: the pairwise-swap local search of balanced_cluster
 * (tree.py:169-198), sequentially exact: D device [n][n] divergences, cid
 * device int64 [n] cluster ids (in/out), rowsum device [n][L] row sums of D
 * over each cluster (in/out), at most `sweeps` passes; sweeps_done
 * (optional, device int32) receives the passes run. */
int fepll_cluster_swap(const double* D, int32_t n, int32_t L, int64_t* cid, double* rowsum,
                       int32_t sweeps, int32_t* sweeps_done, void* stream);

/* debugging: record per-tile pipeline timestamps of one tree level of the
 * warp-specialized scorer into a device buffer (148 x 64 x 8 uint64). */
int fepll_debug_ws_trace(void* device_buffer, int32_t level);
/* debug: ws2 tree-level kernels write globaltimer stamps (CTA entry, after
 * the prologue, end) to device_buffer[depth][148][4] (uint64), the
 * re-scoring kernel its first entry / last exit to element 16*148*4 +
 * 2*depth (+1) (atomic min / max: initialise to ~0 / 0); NULL: off */
int fepll_debug_level_spans(void* device_buffer);

/* Stream-ordered device timestamp: *dst = %globaltimer (nanoseconds) when the
 * stream reaches this point.  A one-thread kernel, so it can be captured in
 * a CUDA graph: restore() replays a captured restore and still fills
 * IterationStats.times (pkg/src/fepll/solver.py:206-254) per call. */
int fepll_stamp(uint64_t* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif
