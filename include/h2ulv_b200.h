/*
 * h2ulv_b200.h — C ABI of the B200-native H²-ULV factorize/solve path.
 *
 * The reference (`h2ulv`, /root/reference/pkg) is pure Python and has no
 * FFI; its dense engine is `dense_core.run_plan` driving LAPACK/BLAS one
 * block at a time (dense_core.py:229-284, called from ulv_factor._run,
 * ulv_factor.py:145-151).  This library replaces that engine: every entry
 * point below executes ONE batched phase of a level (all boxes / all pairs
 * at once) on the GPU.  The Python mirror of the reference API
 * (paper_2502_02395_b200/ulv_factor.py, ulv_solve.py, h2_build.py) binds
 * these symbols through ctypes.
 *
 * Conventions
 *   - all matrices are FP64, row-major (numpy C order): element (r, c) of
 *     a matrix X with leading dimension ld is X[r*ld + c];
 *   - every descriptor array and tile/CTA map passed as `d_*` lives in
 *     device memory; scalars are host values;
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     asynchronous on that stream;
 *   - every function returns 0 on success or a nonzero H2G_E* code; the
 *     message is available from h2g_last_error().  No exception crosses the
 *     ABI.  Numerical breakdown (non-positive pivot) is reported through
 *     the device array `d_npd`, see h2g_chol_panel.
 */
#ifndef H2ULV_B200_H
#define H2ULV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H2G_ABI_VERSION 1

enum {
  H2G_OK = 0,
  H2G_EINVAL = 1,   /* bad argument (null pointer, negative size, ...)   */
  H2G_ECUDA = 2,    /* a CUDA runtime call or launch failed               */
  H2G_ESTEP = 3,    /* unknown step kind in a program                     */
  H2G_ENPD = 4      /* the factorization met a non-positive pivot (status) */
};

/* ---- grouped GEMM ---------------------------------------------------------
 * C = alpha * op(A) * op(B) + beta * C  for every problem of the group.
 * op(A) is M x K, op(B) is K x N.  trans_a / trans_b and the tile shape are
 * uniform for the launch: tile_cfg 2 = 64x64 tiles at 4 CTAs/SM, 7 = 64x64
 * tiles at 3 CTAs/SM (K <= 64 updates), 9 = 32x32 tiles (ragged problems).  flags bit 0 (H2G_GEMM_LOWER, requires
 * M == N) computes only the output tiles on or below the diagonal
 * (SYRK-style Schur updates).  C may alias A when N fits one tile (the
 * in-place TRSM X <- X Linv^T).
 * `tile_start` is the problem's first tile in the launch; d_tile_map[t] is
 * the problem index of tile t (t < total_tiles).
 * Replaces: dense_core.multiply (dense_core.py:84-93) for the phases
 * diag_mul1/2, off_mul1/2 and diag_schur (ulv_factor.py:189-200, 236-259).
 */
#define H2G_GEMM_LOWER 1
typedef struct h2g_gemm_problem {
  const double* A;
  const double* B;
  double* C;
  int32_t M, N, K;
  int32_t lda, ldb, ldc;
  int32_t tile_start;
  int32_t flags;
  double alpha, beta;
} h2g_gemm_problem;

int h2g_gemm_tiles(int M, int N, int flags, int tile_cfg); /* tiles one problem needs */

/* Per-problem extension of a grouped GEMM (h2g_gemm_grouped_ext, NN or NT):
 *   Cin (ld ldcin), when not NULL, is the beta term's source instead of C;
 *   remap_k >= 0 stores a LOWER problem's tile through the compact-WY relabel of
 *   the diag transform (diag_mul1/2, ulv_factor.py:189-200; id_basis's column
 *   order and signs, dense_core.py:140-148): the product is H' = Q^T A Q in
 *   Householder column order (skeleton columns 0..k-1 first, k = remap_k);
 *   entry (a, b), a >= b, goes to H[x][y] (or H[y][x] when x < y) with
 *   x = a - k (a >= k) or a + M - k (a < k), sign-flipped by sgn[a] (a < k)
 *   and sgn[b] (b < k).  Only a >= b is stored, so each lower entry of H has
 *   exactly one writer.  A step carries the ext array in `aux`.
 *   remap_k <= -2 relabels columns only (k = -remap_k - 2): column b of the
 *   product goes to column b - k (b >= k) or b + N - k (b < k), sign-flipped
 *   by sgn[b] (b < k) — q_full = [Q[:, k:] | Q[:, :k] s] from Q = I - Yt Y^T. */
typedef struct h2g_gemm_ext {
  const double* Cin;
  const double* sgn;
  int32_t ldcin;
  int32_t remap_k;  /* >= 0: symmetric relabel; -1: plain store; <= -2: column relabel */
} h2g_gemm_ext;

/* Deterministic split-K for grouped launches under one wave (few-box upper
 * levels): every tile is nsplit consecutive CTAs (the tile map lists each
 * problem's tiles x nsplit CTAs), CTA s accumulates the s-th BK-aligned K
 * range into d_ws, the last CTA of the tile (per-tile counter) sums the
 * partials in the order 0..nsplit-1 and applies alpha / beta — independent of
 * the arrival order.  d_ws: h2g_gemm_split_workspace(tiles, nsplit) bytes,
 * zeroed once (the counters return to zero after every launch).  As a program
 * step: GEMM kind, arg = tile_cfg | nsplit << 8, npd = d_ws.  tile_cfg 2. */
size_t h2g_gemm_split_workspace(int tiles, int nsplit);
int h2g_gemm_grouped_split(int trans_a, int trans_b, int tile_cfg, const h2g_gemm_problem* d_probs,
                           const int32_t* d_tile_map, int total_ctas, int nsplit, void* d_ws, void* stream);

int h2g_gemm_grouped_ext(int trans_a, int trans_b, int tile_cfg, const h2g_gemm_problem* d_probs,
                         const h2g_gemm_ext* d_ext, const int32_t* d_tile_map, int total_tiles, void* stream);
int h2g_gemm_grouped(int trans_a, int trans_b, int tile_cfg, const h2g_gemm_problem* d_probs,
                     const int32_t* d_tile_map, int total_tiles, void* stream);

/* ---- panel step of the partial (ULV) Cholesky --------------------------------
 * For panel q (columns p = 64q .. p+b-1) of every box:
 *   kernel 1, one CTA per descriptor: apply the previous panel's update
 *      (columns p-64 .. p-1, final L; nothing when p == 0) to the diagonal
 *      block, factor it: L_pp -> H, L_pp^-1 -> the 64 x 64 block `Linv`,
 *      pivot status: a pivot that is not > 0 (or NaN) at column p+j records
 *      atomicMin(&d_npd[npd_slot], p+j) — the pivot dpotrf reports as info-1
 *      (dense_core.py:60-63);
 *   kernel 2, one CTA per 64-row chunk of the rows below the panel: apply
 *      the previous panel's update to the chunk rows, then X <- X L_pp^-T.
 * The update of the columns >= p+b+64 by the previous panel (REST) is left
 * to a grouped GEMM issued before this step, so the factorization's critical
 * lane issues two kernels per panel (ulv_factor.py:217-241).  Chunks per
 * box: h2g_chol_panel_tiles (0 when nothing is below); d_tile_map[t] =
 * descriptor of chunk CTA t, tile_start = its first chunk CTA.
 */
typedef struct h2g_chol_panel_desc {
  double* H;          /* n x n, row-major, ld ldh (lower triangle used) */
  double* Linv;       /* 64 x 64 output, ld ldl */
  int32_t ldh, ldl;
  int32_t n;          /* rows of H */
  int32_t p, b;       /* panel start column (multiple of 64) and width (1..64) */
  int32_t npd_slot;
  int32_t tile_start;
  int32_t pad_;
} h2g_chol_panel_desc;

int h2g_chol_panel_tiles(int n, int p, int b);
int h2g_chol_panel(const h2g_chol_panel_desc* d_descs, int count, const int32_t* d_tile_map, int total_tiles,
                   int32_t* d_npd, void* stream);
/* The same step; with d_sync (2 * count + 2 zeroed int32, left zeroed) and
 * count <= h2g_chol_panel_fused_max() (default 128, env H2G_PANEL_FUSED_MAX)
 * it is ONE launch: each CTA takes a ticket, the first `count` factor the
 * diagonal blocks and publish L_pp^-1 through a per-box flag, the rest are
 * the row chunks, which apply the previous panel while the diagonal block is
 * being factored and wait for the flag only before their TRSM. */
int h2g_chol_panel_sync(const h2g_chol_panel_desc* d_descs, int count, const int32_t* d_tile_map, int total_tiles,
                        int32_t* d_npd, int32_t* d_sync, void* stream);
int h2g_chol_panel_fused_max(void);

/* ---- fused per-box partial Cholesky ----------------------------------------
 * ONE CTA per descriptor (box) performs the box's whole elimination
 * (ulv_factor.py:217-241, factor_diag): left-looking over the 64-wide panels
 * of RR, each diagonal block updated by the earlier panels, factored
 * (L_qq -> H, L_qq^-1 -> Linv + 4096 q, pivot status -> d_npd exactly like
 * h2g_chol_panel), every row below it (rest of RR and the SR rows) updated
 * and solved against L_qq^-T in place; then the single Schur update
 * SS -= L(s) L(s)^T on the lower 64 x 64 tiles of the k x k corner.  With Q
 * the rows of V = q_red L^-T (diag_trsm) are formed in the same panel loop.
 * For levels with many boxes: no per-panel launches and no inter-CTA waits.
 */
typedef struct h2g_cholbox_desc {
  double* H;          /* n x n, ld ldh; RR = H[:r, :r], SR = H[r:, :r], SS = H[r:, r:] (lower parts used) */
  double* Linv;       /* ceil(r / 64) blocks of 64 x 64 */
  const double* Q;    /* optional (NULL: none): q_full (n x n, ld ldh) -> V = q_red L^-T ... */
  double* R;          /* ... into R[:, :r] (ld ldh), panel by panel with the rows of H */
  int32_t n, r;
  int32_t ldh, npd_slot;
} h2g_cholbox_desc;

int h2g_chol_box(const h2g_cholbox_desc* d_descs, int count, int32_t* d_npd, void* stream);

/* ---- left-looking row solve --------------------------------------------------
 * X = B L^-T block column by block column, one CTA per 64-row chunk of every
 * descriptor.  For panel q in [q_begin, q_end) (p = 64q, b = min(64, cols-p)):
 *   Xout[r, p:p+b] = (Xin[r, p:p+b] - Xout[r, 0:p] L[p:p+b, 0:p]^T) Linv_q^T
 * with L given by its rows (Lb, ld ldlb, row 0 / column 0) and Linv_q the
 * 64 x 64 inverse of L's q-th diagonal block (at Linv + 4096 q, ld 64).
 * Xin == NULL means B = I (X = L^-T, upper triangular; only rows < p + b are
 * formed).  Xout may equal Xin.  Replaces the tri_solve of
 * V_i = q_red L^-T (dense_core.py:69-81 in diag_trsm, ulv_factor.py:223-234);
 * also forms the root's explicit L^-T used by the solve.
 */
typedef struct h2g_rows_desc {
  const double* Lb;    /* L (cols x cols lower), ld ldlb */
  const double* Xin;   /* rows x cols, ld ldx (or NULL: identity) */
  double* Xout;        /* rows x cols, ld ldx (may equal Xin) */
  const double* Linv;  /* inverses of L's 64 x 64 diagonal blocks, 4096 doubles each */
  const double* pad0_;
  int32_t rows, cols, q_begin, q_end;
  int32_t ldlb, ldx;
  int32_t tile_start;  /* first CTA of this descriptor: ceil(rows / 64) CTAs each */
  int32_t pad1_;
} h2g_rows_desc;

int h2g_trsm_rows(const h2g_rows_desc* d_descs, const int32_t* d_tile_map, int total_tiles, void* stream);

/* ---- block copy / gather ----------------------------------------------------
 * dst[r, c] = src(r, c) for an rows x cols block, where src(r, c) is
 *   mode 0: src[r*lds + c]            (copy)
 *   mode 1: src[c*lds + r]            (transpose)
 *   mode 2: src[max(r,c)*lds + min(r,c)]  (symmetric from the lower half)
 *   mode 3: (r == c) ? 1 : 0              (identity fill; src unused)
 * 64x64 tiles; d_tile_map[t] = descriptor of tile t.
 * Replaces: merge_level / inject_couplings (ulv_factor.py:108-132, 289-303)
 * — the 2x2 assembly of child SS blocks (and far couplings) into the parent
 * near blocks.
 */
typedef struct h2g_copy_desc {
  const double* src;
  double* dst;
  int32_t rows, cols;
  int32_t lds, ldd;
  int32_t mode;
  int32_t tile_start;
} h2g_copy_desc;

int h2g_copy_tiles(int rows, int cols);
int h2g_block_copy(const h2g_copy_desc* d_descs, const int32_t* d_tile_map,
                   int total_tiles, void* stream);

/* ---- substitution ------------------------------------------------------------
 * Vectors are blocks of `w` columns, row-major with leading dimension w.
 *
 * h2g_gemv_grouped: for every output segment o (one CTA each)
 *   y_o = init_o - sum_t op(A_t) x_t           (init_o may alias y_o or be NULL = 0)
 * or, with H2G_GEMV_SPLIT, y = op(A) x written as rows [0, split) -> y and
 * rows [split, m) -> y2 (the basis transform of _transform_in,
 * ulv_solve.py:33-41, split = r).  Terms of output o are
 * d_terms[term_begin .. term_end).  With H2G_GEMV_PLUS the sum is added.
 * A term with A == NULL is the identity (K = m): x_t is added as is.
 * d_chunk_map (optional, NULL = binary search over chunk_start): output index
 * of every chunk.
 * Each output is split into 64-row chunks, one CTA each (chunk_start =
 * running sum of ceil(m / 64)).
 * Replaces the per-box numpy products of _forward/_backward
 * (ulv_solve.py:98-113, 144-181).
 */
#define H2G_GEMV_PLUS 1
#define H2G_GEMV_SPLIT 2
typedef struct h2g_gemv_term {
  const double* A;
  const double* x;
  int32_t lda;
  int32_t trans;   /* 0: A is m x K ; 1: A is K x m (use A^T) */
  int32_t K;
  int32_t pad_;
} h2g_gemv_term;

typedef struct h2g_gemv_out {
  double* y;
  double* y2;        /* SPLIT only */
  const double* init;
  int32_t m;         /* rows of y (before split) */
  int32_t split;     /* SPLIT only */
  int32_t term_begin, term_end;
  int32_t flags;
  int32_t chunk_start; /* first 64-row chunk (CTA) of this output */
} h2g_gemv_out;

int h2g_gemv_grouped(const h2g_gemv_out* d_outs, int n_outs, const h2g_gemv_term* d_terms,
                     const int32_t* d_chunk_map, int total_chunks, int w, void* stream);

/* h2g_xform_t: [y1; y2] = Q^T x for every box (Q n x n row-major, ld ldq;
 * x n x w, ld w; rows [0, split) of the result -> y1, rows [split, n) -> y2):
 * the basis transform of the forward sweep (_transform_in,
 * ulv_solve.py:33-41).  One CTA per 128 output columns of a box (d_tile_map[t]
 * = descriptor of CTA t, tile_start = its first CTA); the rows are split over
 * the CTA's warps.  vec16 != 0 promises every Q row start 16-byte aligned
 * (even ldq, aligned Q) and selects 16-byte loads.
 */
typedef struct h2g_xform_desc {
  const double* Q;
  const double* x;
  double* y1;
  double* y2;
  int32_t n, split, ldq, tile_start;
} h2g_xform_desc;

int h2g_xform_t(const h2g_xform_desc* d_descs, const int32_t* d_tile_map, int total_tiles, int w, int vec16,
                void* stream);

/* h2g_xform_n: out = Q [xr; xs] for every box (Q n x n row-major, ld ldq; xr
 * the first r entries, xs the other n - r, each n x w / ld w; n <= 4096): the
 * basis transform of the backward sweep, full_i = q_red x_R + q_skel x_S
 * (ulv_solve.py:178-181).  One CTA per h2g_xform_n_rows() output rows
 * (d_tile_map as above); vec16 as for h2g_xform_t; max_n = the largest n of
 * the launch (sizes the shared x staging; the step carries it in d0).
 */
typedef struct h2g_xform_n_desc {
  const double* Q;
  const double* xr;
  const double* xs;
  double* out;
  int32_t n, r, ldq, tile_start;
} h2g_xform_n_desc;

int h2g_xform_n(const h2g_xform_n_desc* d_descs, const int32_t* d_tile_map, int total_tiles, int w, int vec16,
                int max_n, void* stream);
int h2g_xform_n_rows(void);

/* h2g_trsv_batched: x_i <- L_i^-1 x_i (trans=0) or L_i^-T x_i (trans=1) for
 * every box, one CTA per box; L_i is the lower r_i x r_i factor stored with
 * leading dimension ldl, Linv the inverses of its 64 x 64 diagonal blocks
 * (h2g_tri_inv / h2g_chol_panel layout, 64*64 doubles per block, block q at
 * Linv + q*4096) (dense_core.tri_solve, dense_core.py:69-81).
 */
typedef struct h2g_trsv_desc {
  const double* L;
  const double* Linv;
  double* x;
  int32_t n;
  int32_t ldl;
} h2g_trsv_desc;

int h2g_trsv_batched(const h2g_trsv_desc* d_descs, int count, int trans, int w, void* stream);

/* ---- complementary basis: batched Householder QR ----------------------------
 * Blocked Householder QR of Z_i (n_i x k_i, in place) in panels of <= 32
 * columns, LAPACK conventions (dgeqrf/dlarfg).  h2g_qr_panel factors the
 * panel Z[p:n, p:p+b] of every box in place (R on/above the diagonal,
 * reflectors below with implicit unit diagonal), copies the reflectors with
 * their unit diagonal into V[p:n, p:p+b], writes tau[p..p+b) and the b x b
 * upper-triangular block factor T (H_p...H_{p+b-1} = I - V T V^T), so that
 * the trailing update (C -= V T^T V^T C) and the explicit formation of Q
 * (Q <- Q - V T V^T Q, last panel first) are h2g_gemm_grouped calls.
 * Replaces: np.linalg.qr(z, mode="complete") in id_basis
 * (dense_core.py:136-144), i.e. the ① complementary basis.
 */
typedef struct h2g_qr_panel_desc {
  double* Z;         /* n x k, ld ldz */
  double* V;         /* explicit reflectors, same layout as Z (zero-initialised) */
  double* tau;       /* length >= k */
  double* T;         /* 32 x 32 block factor for this panel, ld 32 */
  int32_t n, ldz;
  int32_t p, b;
} h2g_qr_panel_desc;

int h2g_qr_panel(const h2g_qr_panel_desc* d_descs, int count, int max_rows, void* stream);  /* max_rows >= max(n - p): panels that fit are factored in shared memory */

/* h2g_basis_finish: given Q (n x n, explicit) and the factored Z (R in the
 * upper triangle), apply the sign convention of id_basis
 * (dense_core.py:140-144): s = sign(diag R[:k,:k]) (0 -> +1),
 * Q[:, :k] *= s, and frame = s[:,None] * R[:k, :] (k x k).  Then reorder the
 * columns of Q into q_full = [q_red | q_skel] in place order.
 */
typedef struct h2g_basis_desc {
  const double* Q;   /* n x n explicit Householder product (input) */
  const double* Z;   /* factored Z (R upper), ld ldz */
  double* qfull;     /* n x n output = [q_red | q_skel] */
  double* frame;     /* k x k output */
  int32_t n, k, ldz;
  int32_t pad_;
} h2g_basis_desc;

int h2g_basis_finish(const h2g_basis_desc* d_descs, int count, void* stream);

/* ---- kernel matrix blocks ------------------------------------------------------
 * out[a, b] = K(|x_rows[a] - x_cols[b]|) with K = 1/r (laplace) or
 * exp(-decay r)/r (yukawa) or exp(-decay r^2) (family 2, the opt-in Gaussian
 * covariance of BASELINE configs[3], decay = 1/l^2); out = shift where the two global point ids are
 * equal (kernels.gen_block, kernels.py:46-64).  Coincident distinct points
 * set d_coincident[0] = 1 (the host then locates the pair and raises
 * CoincidentPointsError like kernels.py:55-57).
 */
typedef struct h2g_kblock_desc {
  const int64_t* rows;
  const int64_t* cols;
  double* out;
  int32_t m, n, ldo;
  int32_t tile_start;
} h2g_kblock_desc;

int h2g_kernel_blocks(const h2g_kblock_desc* d_descs, const int32_t* d_tile_map, int total_tiles,
                      const double* d_points, int family, double shift, double decay,
                      int64_t* d_coincident, void* stream);

/* ---- direct-sum exact-kernel product -------------------------
 * y = A x for the EXACT kernel matrix of n points (row-major n x 3, the
 * cloud's tree order): A_ij = K(|p_i - p_j|) for i != j with the families of
 * h2g_kernel_blocks, A_ii = shift (oracle.dense_assemble + a dense product,
 * oracle.py:34-64, without forming A).  x, y row-major n x nrhs.
 * d_work >= h2g_direct_matvec_workspace(n) doubles (current device); the
 * partial sums are reduced in a fixed order, so y is deterministic.  A
 * second point at distance 0 from any point sets d_coincident[0] = 1
 * (CoincidentPointsError on the host).  Two launches per 4 columns.
 */
int64_t h2g_direct_matvec_workspace(int64_t n);
int h2g_direct_matvec(const double* d_points, const double* d_x, double* d_y, int64_t n, int nrhs, int family,
                      double shift, double decay, double* d_work, int64_t work_elems, int64_t* d_coincident,
                      void* stream);

/* ---- single-block API support (dense_core.cholesky / tri_solve) -------------
 * h2g_sym_check: one CTA per matrix; d_out[2q] = max_{i>j} |A_ij - A_ji|,
 * d_out[2q+1] = max |A_ij| as IEEE bit patterns (non-negative doubles; NaN
 * propagates into the first).  The caller raises the reference's
 * ValueError when the first exceeds 1e-10 x the second
 * (dense_core.py:56-59).
 * h2g_tri_inv: inverses of the 64 x 64 diagonal blocks of lower-triangular
 * L (n x n, ld ldl) in the Linv layout of the Cholesky panels (block q at
 * Linv + 4096 q, ld 64, identity beyond n), so h2g_trsm_rows can solve
 * against any triangular factor; the first zero diagonal entry j records
 * atomicMin(&d_status[status_slot], j) (SingularTriangularError,
 * dense_core.py:75-76); Linv == NULL: that check only.  One CTA per diagonal block: d_tile_map[t] =
 * descriptor of block CTA t, tile_start = its first block CTA.
 */
typedef struct h2g_symcheck_desc {
  const double* A;
  int32_t n, lda;
} h2g_symcheck_desc;

typedef struct h2g_triinv_desc {
  const double* L;
  double* Linv;
  int32_t n, ldl;
  int32_t tile_start, status_slot;
} h2g_triinv_desc;

int h2g_sym_check(const h2g_symcheck_desc* d_descs, int count, unsigned long long* d_out, void* stream);
int h2g_tri_inv(const h2g_triinv_desc* d_descs, const int32_t* d_tile_map, int total_tiles, int32_t* d_status,
                void* stream);

/* ---- native executor ---------------------------------------------------------
 * A factorization is a static list of steps (one batched phase each); the
 * executor issues them back to back on `stream` without returning to
 * Python, optionally captured once into a CUDA graph and replayed.
 */
enum {
  H2G_STEP_GEMM_NN = 0,
  H2G_STEP_GEMM_NT = 1,
  H2G_STEP_GEMM_TN = 2,
  H2G_STEP_GEMM_TT = 3,
  /* 4: retired (the stand-alone diagonal-block step of round 1) */
  H2G_STEP_COPY = 5,
  H2G_STEP_MEMCPY = 6,   /* descs = dst, map = src (bytes in count) */
  H2G_STEP_QR_PANEL = 7,
  H2G_STEP_BASIS = 8,
  H2G_STEP_GEMV = 9,     /* descs = outs, map = terms, grid = chunks, arg = w */
  H2G_STEP_TRSV = 10,    /* descs = trsv descs, grid = w, arg = trans      */
  H2G_STEP_NOP = 12,     /* no kernel: carries a lane's event wait / record  */
  H2G_STEP_CHOL_PANEL = 13, /* descs/map = chol panel descs/tile map; npd = status */
  H2G_STEP_TRSM_ROWS = 14,  /* descs/map = rows descs/tile map */
  H2G_STEP_SYMCHECK = 15,   /* descs = symcheck descs; aux = device output (2 x count u64) */
  H2G_STEP_TRIINV = 16,     /* descs/map = triinv descs/tile map; npd = status */
  H2G_STEP_CHOL_BOX = 17,   /* descs = cholbox descs; npd = status */
  H2G_STEP_XFORM_T = 18,    /* descs/map = xform descs/tile map; arg = w; count < 0: 16-byte loads */
  H2G_STEP_XFORM_N = 19,    /* descs/map = xform_n descs/tile map; arg = w; count < 0: 16-byte loads */
  H2G_STEP_KBLOCK = 11   /* descs/map = kblock descs/tile map; aux = points,
                            npd = coincident flag; arg = family; shift/decay
                            in the two doubles                              */
};

typedef struct h2g_step {
  int32_t kind;
  int32_t count;      /* problems / descriptors (bytes for MEMCPY) */
  int32_t grid;       /* tiles or CTAs (w for GEMV/TRSV) */
  int32_t arg;        /* GEMM: tile_cfg; TRSV: trans; KBLOCK: family; GEMV: w */
  const void* descs;  /* device descriptor array */
  const int32_t* map; /* device tile / CTA map */
  int32_t* npd;       /* PANEL: device pivot-status array */
  const void* aux;    /* KBLOCK: device points (N x 3); GEMV: chunk -> output map */
  double d0, d1;      /* KBLOCK: shift, decay; XFORM_N: d0 = largest box n */
  int32_t lane;       /* 0: the caller's stream, 1..4: the context's side streams */
  int32_t wait_ev;    /* event index to wait on before the step, or -1 */
  int32_t rec_ev;     /* event index to record after the step, or -1 */
  int32_t pad_;
} h2g_step;

/* Execution context of a multi-lane program: four side streams (lanes 1..4)
 * and n_events events.  The factorization uses lane 0 for the critical
 * chain (diagonal transform, Cholesky panels, merge), lane 1 for the
 * look-ahead trailing updates, lane 4 for the V ride-along, lane 2 for the
 * chain-independent off-diagonal skeleton products and lane 3 for the
 * deferred off-diagonal factor blocks (only the solve reads them).  With ctx == NULL every step runs
 * on `stream` in order. */
int h2g_exec_ctx_create(int n_events, void** ctx_out);
int h2g_exec_ctx_destroy(void* ctx);
int h2g_run_program(const h2g_step* steps, int nsteps, void* stream, void* ctx);
/* Serialized run (lanes ignored) with a CUDA event recorded on `stream`
 * before every step and after the last; synchronizes and writes the per-step
 * device time (ms) to out_ms[nsteps] (host array).  Used by bench.py for the
 * per-kernel roofline numbers. */
int h2g_run_program_timed(const h2g_step* steps, int nsteps, void* stream, float* out_ms);
int h2g_graph_capture(const h2g_step* steps, int nsteps, void* stream, void* ctx, void** exec_out);
int h2g_graph_launch(void* exec, void* stream);
int h2g_graph_destroy(void* exec);

/* ---- factorization session (handle-level entry) -------------------------------
 * A session owns one planned factorization: its step program (planned once by
 * the host for a structure, e.g. paper_2502_02395_b200.ulv_factor.FactorPlan,
 * which also owns the device buffers the descriptors point into), captured
 * into a CUDA graph with its own lanes, plus the device pivot-status array
 * (one int32 per box of every level and the root, INT32_MAX = no failure;
 * the program resets it first).  Levels are numbered like the reference:
 * level l holds 2^l boxes, its statuses start at slot_base[l] (l = 0 is the
 * root, one slot).
 *   h2g_session_factor_async: enqueue one factorization on `stream`.
 *   h2g_session_status: wait for it and decode the statuses the way the
 *     reference reports a breakdown — the deepest failing level first, the
 *     first failing box of it — into *status; returns H2G_ENPD when a pivot
 *     failed (NotPositiveDefiniteError(pivot, level, box), dense_core.py:60-63,
 *     ulv_factor.py:218), H2G_OK otherwise.
 */
typedef struct h2g_npd_status {
  int32_t failed;
  int32_t pivot, level, box;
} h2g_npd_status;

int h2g_session_create(const h2g_step* steps, int nsteps, int n_events, int32_t* d_npd, int depth,
                       const int32_t* slot_base, void* stream, void** session_out);
int h2g_session_factor_async(void* session, void* stream);
int h2g_session_status(void* session, void* stream, h2g_npd_status* status);
int h2g_session_destroy(void* session);

int h2g_abi_version(void);
const char* h2g_last_error(void);
int h2g_device_sm_count(void);

#ifdef __cplusplus
}
#endif
#endif /* H2ULV_B200_H */
