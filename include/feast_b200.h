/*
 * feast_b200.h — C ABI of libfeastb200.so, the B200 (sm_100a) FEAST hot path.
 *
 * Plain pointers and sizes only: every matrix argument is a DEVICE pointer to
 * row-major FP64 data; complex matrices are PLANAR (separate re / im planes
 * with the same leading dimension).  A NULL imaginary pointer means "real
 * operand".  All calls are ordered on the context's CUDA stream; functions
 * that return a host-visible result (bad pivot column, Cholesky failure
 * index, reduced-solver status) synchronise that stream.  Status codes:
 *   0 ok, -1 allocation failure (info -1), -2 exactly singular pivot (info -2),
 *   -3 reduced eigensolver failure (info -3), -10 bad argument, -11 CUDA error
 *   (fb_ctx_last_error() has the message).
 * One host thread per context; contexts are independent (one per GPU rank).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/feastlib).
 */
#ifndef FEAST_B200_H
#define FEAST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_ABI_VERSION 1

typedef struct fb_ctx fb_ctx;

int fb_abi_version(void);
/* device: CUDA ordinal; stream: cudaStream_t (NULL = legacy default stream) */
int fb_ctx_create(int device, void* stream, fb_ctx** out);
int fb_ctx_destroy(fb_ctx* ctx);
int fb_ctx_set_stream(fb_ctx* ctx, void* stream);
int fb_ctx_synchronize(fb_ctx* ctx);
const char* fb_ctx_last_error(const fb_ctx* ctx);
/* number of kernels this context has launched (instrumentation for bench.py) */
int64_t fb_ctx_launch_count(const fb_ctx* ctx);

/* ---- dense backend: _DenseOps (dense.py:91-117) ------------------------- */

/* S = z*B - A, B == NULL -> identity.  Replaces the shift formation of
 * _DenseOps.factorize (dense.py:97-103). */
int fb_dense_shift(fb_ctx* ctx, int n, double z_re, double z_im,
                   const double* a_re, const double* a_im, int64_t lda,
                   const double* b_re, const double* b_im, int64_t ldb,
                   double* s_re, double* s_im, int64_t lds);

/* Doubles needed for the per-factor diagonal-block inverses. */
size_t fb_zgetrf_dinv_doubles(int n);

/* In-place LU with partial pivoting of the planar n x n matrix.  piv[n]
 * (device int32): piv[k] = row interchanged with k at step k, 0-based.
 * info (device int32): set to INT32_MAX on entry by this call; on completion
 * holds INT32_MAX, or 1 + the first column with an exactly zero pivot.
 * Asynchronous; read info with fb_read_info.  Replaces lu_factor
 * (dense.py:30-50). */
int fb_zgetrf(fb_ctx* ctx, int n, double* lu_re, double* lu_im, int64_t ld,
              int* piv, double* dinv, int* info);

/* Synchronise and read a device info word; returns -2 and sets *bad_col to
 * the 0-based column when the factorization hit a zero pivot, else 0 and
 * *bad_col = -1.  (SingularMatrixError, dense.py:42-43.) */
int fb_read_info(fb_ctx* ctx, const int* info, int* bad_col);

/* Solve A X = B (adjoint = 0) or A^H X = B (adjoint = 1) in place on the
 * planar n x nrhs block X (ldx).  Replaces lu_solve (dense.py:53-88). */
int fb_zgetrs(fb_ctx* ctx, int n, int nrhs, const double* lu_re, const double* lu_im,
              int64_t ld, const int* piv, const double* dinv, int adjoint,
              double* x_re, double* x_im, int64_t ldx);

/* ---- batched over contour points -------------------------------------- *
 * The Ne shifted systems of one contour pass are independent (the reference
 * pre-factorizes them concurrently with parallel_contour, _driver.py:46-54).
 * These entry points process a strided batch of `count` shifts in one call:
 * item b uses (re, im) + b*lu_stride, piv + b*piv_stride, dinv +
 * b*dinv_stride, info[b], rhs + b*b_stride, x + b*x_stride (strides in
 * elements; a zero rhs stride shares one right-hand-side block).  Each item
 * is computed exactly as by the single-shift call. */

/* S_b = z_b*B - A for count shifts (z_re/z_im are HOST arrays, count <= 64). */
int fb_dense_shift_batched(fb_ctx* ctx, int count, int n, const double* z_re, const double* z_im,
                           const double* a_re, const double* a_im, int64_t lda,
                           const double* b_re, const double* b_im, int64_t ldb,
                           double* s_re, double* s_im, int64_t lds, int64_t s_stride);

int fb_zgetrf_batched(fb_ctx* ctx, int count, int n, double* lu_re, double* lu_im, int64_t ld,
                      int64_t lu_stride, int* piv, int64_t piv_stride, double* dinv,
                      int64_t dinv_stride, int* info);

/* Synchronise and read count info words; bad_cols[b] = -1 or the zero-pivot column. */
int fb_read_info_batched(fb_ctx* ctx, int count, const int* info, int* bad_cols);

/* X_b = op(A_b)^{-1} B_b for every item (out of place). */
int fb_zgetrs_batched(fb_ctx* ctx, int count, int n, int nrhs, const double* lu_re, const double* lu_im,
                      int64_t ld, int64_t lu_stride, const int* piv, int64_t piv_stride,
                      const double* dinv, int64_t dinv_stride, int adjoint,
                      const double* b_re, const double* b_im, int64_t ldb, int64_t b_stride,
                      double* x_re, double* x_im, int64_t ldx, int64_t x_stride);

/* ---- RCI-kernel arithmetic (kernel.py) ---------------------------------- */

/* Counter-based SplitMix64 start block: out(i, j) = U(seed, offset + j*n + i)
 * (numpy order="F" reshape), imaginary plane from offset_im.  Bit-exact with
 * random_uniform (kernel.py:90-102, 496-498, 521-525). */
int fb_splitmix(fb_ctx* ctx, uint64_t seed, int64_t offset_re, int64_t offset_im,
                int n, int m, double* out_re, double* out_im, int64_t ld);

/* Quadrature accumulation (accumulate_subspace, kernel.py:108-124).
 * variant 0 'symmetric':         q -= (w/2) Re(r e^{i theta} x)   (q real)
 * variant 1 'hermitian-direct':  q -= (w/4) r e^{+i theta} x
 * variant 2 'hermitian-adjoint': q -= (w/4) r e^{-i theta} x */
int fb_accumulate(fb_ctx* ctx, int variant, int n, int m,
                  const double* x_re, const double* x_im, int64_t ldx,
                  double* q_re, double* q_im, int64_t ldq,
                  double weight, double radius, double theta);

/* All quadrature terms of one contour pass in one sweep over Q (the
 * accumulate_subspace calls of kernel.py:350-364 / 500-503 / 527-531 for every
 * point of the pass, in the given order): term k is fb_accumulate's update
 * with (variant[k], w[k], radius, theta[k]) on the solve result
 * (x_re[k], x_im[k]) (host array of device pointers, common ldx).  Bitwise
 * equal to calling fb_accumulate term by term; Q is read and written once.
 * count <= 64; variants must be all 0 or all in {1, 2}. */
int fb_accumulate_terms(fb_ctx* ctx, int count, const int* variant, const double* weight,
                        double radius, const double* theta,
                        const double* const* x_re, const double* const* x_im,
                        int n, int m, int64_t ldx,
                        double* q_re, double* q_im, int64_t ldq);

/* C = alpha op(A) op(B) + beta C on planar / real FP64 (DMMA tensor pipe).
 * op: 'N', 'T' or 'C'.  Used for the dense multiplies (dense.py:111-117),
 * projections Q^H A Q, Q^H B Q (kernel.py:377-379) and the Ritz products
 * (kernel.py:411-413). */
int fb_gemm(fb_ctx* ctx, int is_complex, char opa, char opb, int m, int n, int k,
            double alpha_re, double alpha_im,
            const double* a_re, const double* a_im, int64_t lda,
            const double* b_re, const double* b_im, int64_t ldb,
            double beta_re, double beta_im,
            double* c_re, double* c_im, int64_t ldc);

/* M <- (M + M^H)/2 in place (kernel.py:380-381). */
int fb_symmetrize(fb_ctx* ctx, int m, double* re, double* im, int64_t ld);

/* res_j = ||AX_j - lam_j BX_j||_1 / ||scale BX_j||_1, +inf on a zero
 * denominator (_column_residuals, kernel.py:147-153).  lam/res on device. */
int fb_residuals(fb_ctx* ctx, int n, int m, const double* ax_re, const double* ax_im,
                 const double* bx_re, const double* bx_im, int64_t ld,
                 const double* lam, double scale, double* res);
/* The same sums without the division, for a ROW BLOCK of AX / BX (the
 * multi-GPU path shards the rows of _column_residuals, kernel.py:147-153,
 * over ranks and adds the blocks' sums with one all-reduce):
 * sums[2j] = sum_i |AX_ij - lam_j BX_ij|, sums[2j+1] = sum_i |scale BX_ij|. */
int fb_residual_sums(fb_ctx* ctx, int n, int m, const double* ax_re, const double* ax_im,
                     const double* bx_re, const double* bx_im, int64_t ld,
                     const double* lam, double scale, double* sums);

/* Cholesky probe of the leading m x m block: *fail = 0 or the 1-based index of
 * the first non-positive pivot (spd_factor, reduced.py:22-40).  Synchronous. */
int fb_chol_check(fb_ctx* ctx, int m, const double* b_re, const double* b_im, int64_t ld,
                  int* fail);

/* Reduced eigenproblem aq phi = eps bq phi (generalized_eig, reduced.py:188-218):
 * eps[m] ascending (device), phi planar m x m (ldphi), *status = 0 ok, else
 * the solve failed (info -3).  Synchronous. */
int fb_reduced_eig(fb_ctx* ctx, int m, const double* aq_re, const double* aq_im,
                   const double* bq_re, const double* bq_im, int64_t ld,
                   double* eps, double* phi_re, double* phi_im, int64_t ldphi, int* status);

/* interleaved complex128 (ldz complex elements) <-> planar */
int fb_pack(fb_ctx* ctx, int n, int m, const double* z, int64_t ldz,
            double* re, double* im, int64_t ld, int to_planar);

/* ---- banded backend: _BandedOps (banded.py:149-178) --------------------- */

/* Band layouts (device, row-major by band row):
 *   fb   : (2kl+1) x n full band, row kl+s = s-th subdiagonal (expand_band,
 *          banded.py:21-47); real (fb_im NULL) or planar complex.
 *   fact : (3kl+1) x n planar complex LU working array + ipiv[n]
 *          (band_lu_factor, banded.py:68-103, kv = 2kl). */

/* y = FB x for an n x m block (band_matvec, banded.py:50-65). */
int fb_band_matvec(fb_ctx* ctx, int n, int kl, int m,
                   const double* fb_re, const double* fb_im, int64_t ldb,
                   const double* x_re, const double* x_im, int64_t ldx,
                   double* y_re, double* y_im, int64_t ldy);

/* fact = LU(z*FB - FA) (banded.py:156-164 + 68-103).  FB NULL -> identity.
 * info as fb_zgetrf. */
int fb_band_factor(fb_ctx* ctx, int n, int kl, double z_re, double z_im,
                   const double* fa_re, const double* fa_im,
                   const double* fb_re, const double* fb_im, int64_t ldb,
                   double* fact_re, double* fact_im, int* ipiv, int* info);

/* In-place band solve, direct or adjoint (band_lu_solve, banded.py:106-146). */
int fb_band_solve(fb_ctx* ctx, int n, int kl, int nrhs,
                  const double* fact_re, const double* fact_im, const int* ipiv,
                  int adjoint, double* x_re, double* x_im, int64_t ldx);

/* Partitioned (SPIKE) band path, batched over count shifts (count <= 64,
 * 1 <= kl <= 16).  Replaces the per-shift _BandedOps.factorize / solve
 * (banded.py:156-170) for the whole contour: the band is cut into partitions
 * factored independently (pivoting inside partitions) and coupled through a
 * small interface system.  Per shift b: fact (3kl+1) x n planar at
 * fact + b*fact_stride, ipiv[n] at ipiv + b*ipiv_stride, aux at
 * aux + b*aux_stride (fb_band_aux_doubles(n, kl) doubles). */
int64_t fb_band_aux_doubles(int n, int kl);
int fb_band_factor_batched(fb_ctx* ctx, int count, int n, int kl, const double* z_re, const double* z_im,
                           const double* fa_re, const double* fa_im,
                           const double* fb_re, const double* fb_im, int64_t ldb,
                           double* fact_re, double* fact_im, int64_t fact_stride,
                           int* ipiv, int64_t ipiv_stride, double* aux, int64_t aux_stride, int* info);
/* In place: X_b <- S(z_b)^-1 X_b (direct solve only; the Hermitian banded
 * driver serves A^H solves from the factor of conj(z), S(z)^H = S(conj z)). */
int fb_band_solve_batched(fb_ctx* ctx, int count, int n, int kl, int nrhs,
                          const double* fact_re, const double* fact_im, int64_t fact_stride,
                          const int* ipiv, int64_t ipiv_stride, const double* aux, int64_t aux_stride,
                          double* x_re, double* x_im, int64_t ldx, int64_t x_stride);
/* Same solve with the right-hand sides read from Y (y_re/y_im at
 * + b*y_stride; y_stride = 0: one block shared by every shift, e.g. the
 * contour pass's Y; y_im == NULL: real Y) and the solutions written to X
 * (_BandedOps.solve, banded.py:166-170, for all shifts of a pass at once). */
int fb_band_solve_batched_rhs(fb_ctx* ctx, int count, int n, int kl, int nrhs,
                              const double* fact_re, const double* fact_im, int64_t fact_stride,
                              const int* ipiv, int64_t ipiv_stride, const double* aux, int64_t aux_stride,
                              const double* y_re, const double* y_im, int64_t ldy, int64_t y_stride,
                              double* x_re, double* x_im, int64_t ldx, int64_t x_stride);

/* One whole contour pass of the banded drivers (kernel.py:350-364 with
 * _BandedOps.solve, banded.py:166-170, and accumulate_subspace,
 * kernel.py:108-124): every resident shift b is solved against the pass's
 * right-hand side Y (shared by all shifts; y_im NULL: real Y) and the nterms
 * quadrature terms -- term t uses the solve of shift item[t] with
 * (variant[t], w[t], theta[t]) as fb_accumulate -- are folded into Q in the
 * given order.  The spike correction of the partitioned solve is applied
 * inside the accumulation kernel (FP64 tensor pipe), so the corrected
 * solutions are never written: X is work space of count blocks and ends
 * holding the uncorrected partition solves. */
int fb_band_solve_accumulate(fb_ctx* ctx, int count, int n, int kl, int nrhs,
                             const double* fact_re, const double* fact_im, int64_t fact_stride,
                             const int* ipiv, int64_t ipiv_stride, const double* aux, int64_t aux_stride,
                             const double* y_re, const double* y_im, int64_t ldy,
                             double* x_re, double* x_im, int64_t ldx, int64_t x_stride,
                             int nterms, const int* item, const int* variant, const double* w, double r,
                             const double* theta, double* q_re, double* q_im, int64_t ldq);

/* ---- CSR backend (feast_scsr / feast_hcsr, sparse.py:430-517) ---------- */
/* Y = M X for a full-pattern CSR matrix M (0-based int64 indptr[n+1] /
 * indices[nnz], values planar: val_im NULL for real M) and a row-major
 * n x m block X (x_im NULL: real).  Replaces _csr_block_matvec
 * (sparse.py:156-169) behind _SparseOps.multiply_a / multiply_b
 * (sparse.py:454-462).  y_im is required when M or X is complex.
 * row_order (NULL: 0..n-1) is the order rows are visited in -- a
 * bandwidth-reducing permutation keeps the gathered X rows L2-resident;
 * results do not depend on it. */
int fb_csr_matvec(fb_ctx* ctx, int n, int m, const int64_t* indptr, const int64_t* indices,
                  const double* val_re, const double* val_im,
                  const double* x_re, const double* x_im, int64_t ldx,
                  double* y_re, double* y_im, int64_t ldy, const int64_t* row_order);
/* dst(i, :) = src(perm[i], :) for i < n (row gather; src_im and dst_im both
 * NULL for real blocks).  Carries right-hand sides into and out of the
 * bandwidth-reducing order of the CSR direct solver (the role of
 * _SparseSymbolic.perm, sparse.py:209-212 and 292, 312-313). */
int fb_permute_rows(fb_ctx* ctx, int n, int m, const int64_t* perm,
                    const double* src_re, const double* src_im, int64_t lds,
                    double* dst_re, double* dst_im, int64_t ldd);
/* Lockstep diagonal-preconditioned BiCGStab over all m columns of B
 * (_bicgstab + _IterativeFactor._solve_with, sparse.py:354-427): solves
 * S X = B with S the full CSR (indptr/indices 0-based int64, planar complex
 * values s_re/s_im) and d its diagonal (zeros replaced by 1).  b (real when
 * b_im NULL) and x are row-major planar blocks; ldx must equal ld.
 * phase 0 initialises (x = 0, r = rhat = b, per-column |b|); phase 1 runs
 * `iters` more iterations and then writes istate[2m] = columns still
 * iterating, istate[2m+1] = first failure code (0 none; -1 rho = 0,
 * -2 rhat.v = 0, -3 t.t = 0, -4 maxiter reached: the reference's
 * SingularMatrixError cases).  istate holds 2m+2 ints; work holds
 * fb_bicgstab_workspace_doubles(n, m, ld) doubles.  row_order (NULL: natural)
 * is the SpMM row visiting order, as in fb_csr_matvec; it never changes
 * results. */
int64_t fb_bicgstab_workspace_doubles(int n, int m, int64_t ld);
int fb_bicgstab(fb_ctx* ctx, int phase, int n, int m, const int64_t* indptr, const int64_t* indices,
                const double* s_re, const double* s_im, const double* d_re, const double* d_im,
                const double* b_re, const double* b_im, int64_t ldb, double* x_re, double* x_im, int64_t ldx,
                double tol, int maxiter, int iters, double* work, int64_t ld, int* istate,
                const int64_t* row_order);

#ifdef __cplusplus
}
#endif

#endif /* FEAST_B200_H */
