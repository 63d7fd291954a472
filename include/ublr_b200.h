/* ublr_b200.h — C ABI of the B200 (sm_100a) uBLR compression hot path.
 *
 * Drop-in boundary for the matrix-free uniform-BLR compressor of
 * arXiv 2501.05528 (reference: /root/reference/pkg/src/ublr, "ref/" below).
 * The reference's compressor entry points stay Python
 * (ref/reconstruction.py:498-687); they call these functions through ctypes
 * (paper_2501_05528_b200/_lib.py). Every function:
 *   - takes DEVICE pointers (fp64 / int32 / int64), explicit sizes and a
 *     cudaStream_t (passed as void*), and allocates nothing itself unless a
 *     workspace argument says so;
 *   - returns UBLR_OK (0) or a negative status; ublr_last_error() gives the
 *     message. The Python layer maps UBLR_ERR_VALUE -> ValueError,
 *     UBLR_ERR_NUMERIC -> numpy.linalg.LinAlgError, UBLR_ERR_CUDA -> RuntimeError.
 *
 * Layout conventions (see DESIGN.md §Data layout):
 *   - points are renumbered block-contiguously: block i owns permuted rows
 *     [off[i], off[i+1]); perm[p] is the original index of permuted row p;
 *   - dense blocks are row-major; sketches Y/Z are N x s row-major in
 *     permuted row order; bases U/V are N x k row-major (block i rows,
 *     columns [0, k_i)); the core is K x K row-major with K = sum k_i;
 *   - near-field blocks B_ij are stored in neighbour-CSR order (which is the
 *     reference's sorted (i, j) order), block p at b_off[p], m_i x m_j
 *     row-major.
 */
#ifndef UBLR_B200_H
#define UBLR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  UBLR_OK = 0,
  UBLR_ERR_VALUE = -1,   /* bad arguments / configuration  -> ValueError      */
  UBLR_ERR_CUDA = -2,    /* CUDA runtime failure           -> RuntimeError    */
  UBLR_ERR_NUMERIC = -3, /* numerical failure              -> LinAlgError     */
  UBLR_ERR_RETRY = -4    /* internal: caller should retry with more workspace */
};

/* Operator kinds for the on-the-fly operator tiles. */
enum { UBLR_OP_DENSE = 0, UBLR_OP_LOG = 1, UBLR_OP_INV = 2 };

/* Operator descriptor: the black-box A of ref/operators.py:24-35, as the
 * GPU sees it. DENSE: A (original order, row-major, lda), gathered through
 * perm (NULL = identity); transpose != 0 means A^T. LOG: A(x,y) = -log|x-y|; INV: 1/|x-y|;
 * the diagonal (same original index) takes `diag`. coords are permuted,
 * structure-of-arrays: coords[a*n + p]. */
typedef struct {
  int32_t kind;
  int32_t dim;
  int32_t transpose;
  int32_t pad_;
  const double* A;
  int64_t lda;
  const int32_t* perm;
  const double* coords;
  int64_t n;
  double diag;
} ublr_op_t;

/* One Gaussian stream of the reference's RandomStream (ref/linalg.py:14-52):
 * numpy Philox4x64-10 with 128-bit key (SeedSequence-derived, host side),
 * counter starting at 0, `standard_normal` ziggurat, row-major fill.
 * Normal n goes to out[out_offset + rowmap[n / cols] * ld + n % cols]
 * (rowmap == NULL means identity). */
typedef struct {
  uint64_t key0, key1;
  int64_t count;
  int64_t cols;
  int64_t ld;
  int64_t out_offset;
  const int32_t* rowmap;
} ublr_rng_stream_t;

const char* ublr_last_error(void);
int ublr_version(void);
int ublr_device_check(void);

/* Philox keys of the reference's RandomStream(seed, key) (ref/linalg.py:30-35:
 * np.random.Philox(SeedSequence(seed, spawn_key=key)), i.e.
 * SeedSequence.generate_state(2, uint64)) for n spawn keys prefix + suffix_s.
 * Host function. `run` = uint32 words of the seed (little-endian, >= 1 word),
 * `prefix` the words shared by all keys, `suffix` n x nsuffix words;
 * keys_out is n x 2 uint64. */
int ublr_seedseq_keys(const uint32_t* run, int nrun, const uint32_t* prefix, int nprefix,
                      const uint32_t* suffix, int nsuffix, int64_t n, uint64_t* keys_out);

/* Null vectors for the tagging plan (ref/tagging.py:126-139, through
 * ref/linalg.py:72-94): for each row set s (CSR ptr/idx into the b x ell
 * tagging matrix T, fewer than ell rows), Z[s] = last column of the complete
 * Householder Q of T[rows]^T and res[s] = ||T[rows] Z[s]||. Host function. */
int ublr_null_vectors(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int nsets, double* Z,
                      double* res);
/* Device twin of ublr_null_vectors (device pointers; every set must have
 * fewer than ell rows, ell <= 32): bitwise the same Z and residuals as the
 * host function (shared explicitly-rounded arithmetic). */
int ublr_null_vectors_device(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int nsets, double* Z,
                             double* res, void* stream);
/* Tagging-plan aspect ratios (ref/tagging.py:110-123): rho[i] = max/min over
 * the far field j of |T[j] . Z[i]| (T, Z: b x ell row-major device arrays;
 * neighbour CSR nptr/nidx), 1 if the max is 0, inf if the min is 0, NaN if
 * the far field is empty. ell <= 32. */
int ublr_tag_aspect(const double* T, const double* Z, int ell, const int32_t* nptr, const int32_t* nidx, int b,
                    double* rho, void* stream);
/* One evaluation of the tagging redraw policy on the host: null vectors Z and
 * residuals res (ublr_null_vectors), scale[i] = max(1, ||T[rows_i]||_F), and
 * (if rho != NULL) the aspect ratios as ublr_tag_aspect. Host pointers. */
int ublr_tag_plan_host(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int b, double* Z,
                       double* res, double* scale, double* rho);

/* K1 — ref/linalg.py:38-52 (`RandomStream.normal` / `gaussian`), called at
 * ref/bases.py:97-98, :163-168, :229-230 and ref/reconstruction.py:405.
 * Bit-compatible with numpy. `streams` is a DEVICE array. Workspace bytes
 * from ublr_rng_workspace_bytes. */
int64_t ublr_rng_workspace_bytes(const int64_t* counts, int n_streams);
int ublr_rng_normals(const ublr_rng_stream_t* streams_dev, const int64_t* counts_host, int n_streams,
                     double* out, void* workspace, int64_t workspace_bytes, void* stream);

/* K2/K3 — tagged sketch, ref/bases.py:163-172 (assemble_tagging_test_matrix +
 * op.apply / op.apply_adjoint). Y[:, c*gc+q] for block-row i accumulates
 * sum_j T[j,c] * (A_ij X_j)[:, q] (Kronecker-restructured: each A tile meets
 * its own test block once). X is N x gc (permuted rows, ld_x); T is b x ell.
 * Computes rows [row_begin, row_end) of Y = A Omega (N x ell*gc, ld_y; Y is
 * indexed by absolute permuted row, so a row shard passes Y - row_begin*ld_y). */
int ublr_sketch_tagged(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                       const double* X, int64_t ld_x, int gc, double* Y, int64_t ld_y, int row_begin,
                       int row_end, void* stream);
/* Both sides of a NON-symmetric tagged sketch in one launch: Y = A Omega
 * (op, test blocks G) and Z = A^T Psi (op_adj = the adjoint descriptor, H),
 * the same tagging matrix T. Replaces two ublr_sketch_tagged calls. */
int ublr_sketch_tagged_two(const ublr_op_t* op, const ublr_op_t* op_adj, const int32_t* off, int b, const double* T,
                           int ell, const double* G, const double* H, int64_t ld_x, int gc, double* Y, double* Z,
                           int64_t ld_y, int row_begin, int row_end, void* stream);
/* Symmetric operator: [Y | Z] = A [Omega | Psi] in one pass over A. */
int ublr_sketch_tagged_pair(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                            const double* G, const double* H, int64_t ld_x, int gc,
                            double* Y, double* Z, int64_t ld_y, int row_begin, int row_end, void* stream);
/* The same products with a COMPENSATED fold over the column blocks: the
 * rounding error of every Y_c += T[j,c] (A_ij X_j) is recovered exactly and
 * summed apart. Type B (ref/reconstruction.py:326-376,
 * tagging_pinv_discrepancy) divides pair-combined sketches by projected tags
 * as small as 1e-4 and feeds them to the core least squares, so the
 * sketch's fold rounding is the leading term of the B2 approximation error
 * at N = 65,536; type A does not need it. H and Z may both be NULL (one
 * side). ell <= 10; larger ell falls back to the plain fold. */
int ublr_sketch_tagged_comp(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                            const double* G, const double* H, int64_t ld_x, int gc,
                            double* Y, double* Z, int64_t ld_y, int row_begin, int row_end, void* stream);

/* The tagged sketch through a staged strip of A (kernel operators; n and
 * every off[j] even): rows [r0, r0 + R) of A are evaluated once into
 * `workspace` and the sketch kernel's producers only copy tiles, so no FP64
 * evaluation shares the pipe with the DMMAs and A is evaluated once per strip
 * instead of once per 128-column tile. R = ublr_sketch_tagged_staged_rows(n,
 * columns (gc, or 2 gc with H), rows, workspace_bytes); 0 means no strip of
 * that size fills the SMs -- use the entry points above. `compensated` as
 * ublr_sketch_tagged_comp. Same products as the fused entry points. */
int ublr_sketch_tagged_staged_rows(int64_t n, int ncols, int rows, int64_t workspace_bytes);
int ublr_sketch_tagged_staged(const ublr_op_t* op, const int32_t* off, int b, const double* T, int ell,
                              const double* G, const double* H, int64_t ld_x, int gc,
                              double* Y, double* Z, int64_t ld_y, int row_begin, int row_end,
                              int compensated, void* workspace, int64_t workspace_bytes, void* stream);

/* Generic operator apply (ref/operators.py:48-52 and every op.apply call of
 * the pipeline): out (N x w, permuted rows, ld_o) = A X (N x w, ld_x). */
int ublr_apply(const ublr_op_t* op, const double* X, int64_t ld_x, int w, double* out, int64_t ld_o,
               void* stream);
/* The same product for a WIDE right-hand side of a kernel operator (the
 * 2(9m + k + p)-column block-nullification sketch, the K + p - s extra
 * columns of the type-B core): A is evaluated once per strip of rows into
 * `workspace` (any size from one 128-row strip, 128 n doubles, up to
 * ublr_apply_staged_workspace_bytes) and multiplied by all w columns with the
 * stored-operand DMMA GEMM; ublr_apply evaluates it inside the GEMM, once per
 * 256-column tile. Same entries, same result up to summation order. */
int64_t ublr_apply_staged_workspace_bytes(int64_t n, int w);
int ublr_apply_staged_rows(int64_t n, int w, int64_t workspace_bytes);   /* rows per strip; 0 = workspace too small */
int ublr_apply_staged(const ublr_op_t* op, const double* X, int64_t ld_x, int w, double* out, int64_t ld_o,
                      void* workspace, int64_t workspace_bytes, void* stream);

/* K4 — combine + QR: ref/bases.py:174-189, :207-210 with ref/linalg.py:55-69
 * and ref/bases.py:78-83. Per block i: sample S_i (m_i x k) is
 *   mode 0 (tag):   sum_c z[i,c] * Y[rows_i, c*gc + q], q < k;
 *   mode 1 (cols):  Y[rows_i, col0[i] + q]            (naive, bn samples);
 *   mode + 2:       plain QR (no identity shortcut when k >= m_i; col_basis).
 * Q = first k_i columns of the unpivoted Householder QR (LAPACK dlarfg
 * convention) of S_i, or the identity when k >= m_i. Writes U (N x ldu). */
int ublr_block_qr(const double* Y, int64_t ld_y, int mode, const double* z, int ell, int gc,
                  const int32_t* col0, const int32_t* off, int b, int k, double* U, int64_t ld_u,
                  void* stream, int m_max);
/* Both sides of a tagging bases step in one launch: U_i from Y and V_i from
 * Z (mode 0 of ublr_block_qr, the same z^(i)); grid b x 2. */
int ublr_block_qr_pair(const double* Y, const double* Z, int64_t ld_y, const double* z, int ell, int gc,
                       const int32_t* off, int b, int k, double* U, double* V, int64_t ld_u, void* stream,
                       int m_max);

/* K6 — coupling (ref/reconstruction.py:185-198, direct_core):
 * core[roff[i]:, roff[j]:] = U_i^T A_ij V_j for block rows i0 <= i < i1 and all
 * j (U and core indexed by absolute rows: a block-row shard passes shifted
 * pointers). Any block size; effective ranks up to 96 (blocks above 256
 * points or ranks above 64 take the general kernel). */
int ublr_coupling(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k,
                  const double* U, const double* V, int64_t ld_uv, double* core, int64_t ld_c,
                  void* stream, int m_max, int i0, int i1);

/* K7 — near field with the colour-probe semantics of
 * ref/reconstruction.py:201-244: for each near pair p = (i, j),
 *   B_ij[:, q] = sum_{j' in colour(j), q < m_j'} (A_ij' - U_i C_ij' V_j'^T)[:, q]
 * (the same-colour far residuals of block row i leak in).
 * Colour members in CSR (cptr, cidx); pairs given by (pair_i[p], nidx[p]);
 * B block p at B + b_off[p], m_i x m_j row-major. Workspace:
 * ublr_nearfield_workspace_bytes(n_pairs, k, m_max). */
int64_t ublr_nearfield_workspace_bytes(int n_pairs, int k, int m_max);
int ublr_nearfield_colour(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k,
                          const double* U, const double* V, int64_t ld_uv, const double* core,
                          int64_t ld_c, const int32_t* colour, const int32_t* cptr, const int32_t* cidx,
                          int n_colours, int m_max, const int32_t* pair_i, const int32_t* nidx, int n_pairs,
                          const int64_t* b_off, double* B, void* workspace, int64_t workspace_bytes,
                          void* stream);

/* K6 + K7 fused for small blocks (m_max <= 64, effective rank <= 32; configs
 * 1-2): one CTA per (block row i, colour c) writes C_ij = U_i^T A_ij V_j for
 * every j of colour c (as ublr_coupling) and, when block row i has a near pair
 * p = (i, j*) with colour(j*) = c, B_p exactly as ublr_nearfield_colour, from
 * the same generated A_ij (one operator pass instead of two, no workspace).
 * pair_of[i * n_colours + c] = p, or -1 when block row i has no near pair of
 * colour c (a valid colouring has at most one). Rows i0 <= i < i1. */
int ublr_coupling_nearfield(const ublr_op_t* op, const int32_t* off, const int32_t* roff, int b, int k,
                            const double* U, const double* V, int64_t ld_uv, double* core, int64_t ld_c,
                            const int32_t* cptr, const int32_t* cidx, int n_colours, int m_max,
                            const int32_t* pair_of, const int32_t* nidx, const int64_t* b_off, double* B,
                            void* stream, int i0, int i1);

/* K12 — A_hat X (adjoint = 0) or A_hat^T X (adjoint = 1) for the compressed
 * representation (ref/reconstruction.py:93-119): blockwise U C V^T X + B X.
 * tpair[q] for q in the CSR row of j gives the pair index of (nidx[q], j).
 * work: ublr_blr_apply_workspace_bytes(K, w). */
int64_t ublr_blr_apply_workspace_bytes(int64_t K, int w);
int ublr_blr_apply(const double* U, const double* V, int64_t ld_uv, const double* core, int64_t K,
                   const double* B, const int64_t* b_off, const int32_t* off, const int32_t* roff,
                   const int32_t* nptr, const int32_t* nidx, const int32_t* tpair, int b,
                   const double* X, int64_t ld_x, int w, int adjoint, double* out, int64_t ld_o,
                   double* work, void* stream);

/* K12b — exact blockwise Frobenius norms for the parity gates (BASELINE.json;
 * the compressed form is ref/reconstruction.py:50-132). For block rows
 * i0 <= i < i1 and every j: err2[(i-i0)*b + j] = ||A_ij - A_hat_ij||_F^2 and
 * (a2 != NULL) a2[...] = ||A_ij||_F^2, with A_ij generated from the operator
 * descriptor and A_hat_ij = U_i C_ij V_j^T (+ B_ij on near pairs, neighbour
 * CSR nptr/nidx, block p at B + b_off[p]). U and core are indexed by absolute
 * rows (a block-row shard passes shifted pointers); V holds all rows. B may
 * be NULL (no near blocks). Effective ranks from roff; k = max rank <= 96.
 * Deterministic (fixed-order reductions). */
int ublr_frob_error(const ublr_op_t* op, const int32_t* off, const int32_t* nptr, const int32_t* nidx,
                    const int64_t* b_off, int b, const int32_t* roff, int k, const double* U, const double* V,
                    int64_t ld_uv, const double* core, int64_t ld_c, const double* B, int i0, int i1, double* err2,
                    double* a2, void* stream);
/* diff2[(i-i0)*b + j] = ||A_hat1_ij - A_hat2_ij||_F^2 for two compressed
 * representations on the same tessellation (the GPU's own rounding
 * sensitivity, sharded vs single-GPU runs); k1 + k2 <= 96. */
int ublr_frob_diff(const int32_t* off, const int32_t* nptr, const int32_t* nidx, const int64_t* b_off, int b,
                   const int32_t* roff1, int k1, const double* U1, const double* V1, int64_t ld1, const double* core1,
                   int64_t ldc1, const double* B1, const int32_t* roff2, int k2, const double* U2, const double* V2,
                   int64_t ld2, const double* core2, int64_t ldc2, const double* B2, int i0, int i1, double* diff2,
                   void* stream);

/* Batched dense fp64 building blocks (no cuBLAS / cuSOLVER), used by the
 * block-nullification null space (ref/linalg.py:72-94 at ref/bases.py:102-110)
 * and the type-B solves (ref/reconstruction.py:252-421). Row-major;
 * op(A) = A or A^T (ta); amap/bmap (nullable) remap STORAGE rows per batch
 * entry (stride sAm / sBm), so gathered operands such as Omega[nbr(i)] are
 * read in place; cmap remaps C's rows (scatter). C = alpha op(A) op(B) + beta C. */
int ublr_gemm_batched(int ta, int tb, int M, int N, int K, double alpha, const double* A, int64_t lda, int64_t sA,
                      const int32_t* amap, int64_t sAm, const double* B, int64_t ldb, int64_t sB,
                      const int32_t* bmap, int64_t sBm, double beta, double* C, int64_t ldc, int64_t sC,
                      const int32_t* cmap, int64_t sCm, int batch, void* stream);
/* Panel step of a blocked upper Cholesky A = R^T R: factor the nb x nb
 * diagonal block at (j0, j0) of each A_b into R_b and write R11^-1
 * (batch x nb x nb) to Rinv. status != 0 if a block is not positive definite. */
int ublr_potrf_diag(double* A, int64_t lda, int64_t sA, int j0, int nb, double* R, int64_t ldr, int64_t sR,
                    double* Rinv, int* status, int batch, void* stream);
/* Panel step of a blocked no-pivot LU of (W + diag(D)) where D_jj = sign(w_jj)
 * is chosen when column j becomes the pivot (Householder reconstruction sign
 * rule): writes L11\U11 into LU, L11^-1 / U11^-1 (batch x nb x nb) and D. */
int ublr_lu_sign_diag(double* W, int64_t ldw, int64_t sW, int j0, int nb, double* LU, int64_t ldlu, int64_t sLU,
                      double* Linv, double* Uinv, double* D, int64_t sD, int* status, int batch, void* stream);
/* R-scaled variant for the block-nullification null space:
 * the factored matrix is D R - B1^T = (D - Q_top) R with R upper triangular
 * (n x n, batch stride sR). Row j of D R is added when j becomes the pivot
 * row, and after the panel the rows' D R12 (columns j0+nb .. n) are added to
 * W12 so that U12 = L11^-1 W12 follows. L is the L of (D - Q_top); U = U' R^-1.
 * With R == NULL this is ublr_lu_sign_diag. */
int ublr_lu_sign_diag_r(double* W, int64_t ldw, int64_t sW, int j0, int nb, double* LU, int64_t ldlu, int64_t sLU,
                        double* Linv, double* Uinv, double* D, int64_t sD, int* status, const double* R, int64_t ldr,
                        int64_t sR, int n, int batch, void* stream);
/* C_b = alpha A_b^T A_b + beta C_b on the tiles that touch the upper triangle
 * (A_b: K x M row-major; the strictly-lower tiles of C are left untouched,
 * tiles crossing the diagonal are written whole). Symmetric rank-k update of
 * the blocked Cholesky. */
int ublr_syrk_upper_batched(int M, int K, double alpha, const double* A, int64_t lda, int64_t sA, double beta,
                            double* C, int64_t ldc, int64_t sC, int batch, void* stream);
/* out_b[r][c] (or [c][r] with transpose) = src_b[map_b[r] * ld + col0 + c]. */
int ublr_gather(const double* src, int64_t ld, int64_t s_src, const int32_t* map, int64_t s_map, int rows, int cols,
                int col0, int transpose, double* out, int64_t ldo, int64_t s_out, int batch, void* stream);
/* Gram assembly from shared neighbour-pair products: block (a, b) of G_c is
 * P[pid] or P[-pid-1]^T, pid = map[c][a][b] (nb x nb blocks of m x m). */
int ublr_assemble_gram(const double* P, const int32_t* map, int nb, int m, double* G, int batch, void* stream);
/* W_b[r][c] += d_b[r] * R_b[r][c] on a rows x cols block (the D R12 rows of a
 * sign-LU panel, when ublr_lu_sign_diag_r is called with n = j0 + nb). */
int ublr_add_scaled_rows(double* W, int64_t ldw, int64_t s_w, const double* R, int64_t ldr, int64_t s_r,
                         const double* d, int64_t s_d, int rows, int cols, int batch, void* stream);
/* X_b[r][c] *= d_b[r]. */
int ublr_scale_rows(double* X, int64_t ldx, int64_t s_x, const double* d, int64_t s_d, int rows, int cols,
                    int batch, void* stream);

/* Type B (ref/reconstruction.py:326-376): per near pair p = (pair_i[p], .)
 * comb_p[r, q] = sum_c w_p[c] Y[off_i + r, c*gc + q] (w_p = z_p / denominator_p),
 * out is n_pairs x m_max x gc. */
int ublr_tag_combine_pairs(const double* Y, int64_t ld_y, int gc, int ell, const double* w, const int32_t* pair_i,
                           const int32_t* off, int n_pairs, int m_max, double* out, void* stream);
/* Near blocks between the flat neighbour-CSR layout (block p at b_off[p],
 * m_i x m_j row-major) and a padded per-pair layout (block p at
 * p * m_max * m_max, row stride m_max): to_padded = 1 copies flat -> padded,
 * 0 copies padded -> flat. Used by the type-B solves on ragged tessellations. */
int ublr_pairs_pad(double* flat, const int64_t* b_off, const int32_t* pair_i, const int32_t* nidx, const int32_t* off,
                   int n_pairs, int m_max, double* padded, int to_padded, void* stream);
/* Explicit tagged test matrix Omega[r, c*gc + q] = T[block(r), c] G[r, q]
 * (ref/bases.py:126-137), permuted rows. */
int ublr_assemble_tagged(const double* T, int ell, const double* G, int64_t ld_g, int gc, const int32_t* off, int b,
                         double* out, int64_t ld_o, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UBLR_B200_H */
