// Dense shifted complex LU with partial pivoting and its multi-RHS solves.
//
// Restates feastlib's dense backend (dense.py:30-88, _DenseOps dense.py:91-117)
// as a blocked algorithm for sm_100a:
//   * shift formation S = z B - A (dense.py:97-103), planar complex;
//   * right-looking blocked LU, outer block NB = 128 (trailing update is one
//     DMMA ZGEMM with K = 128), inner sub-panels of PW = 32 columns;
//   * each sub-panel is factored by ONE kernel that keeps the panel rows
//     resident in shared memory and exchanges one (|pivot|, row, row-data)
//     record per CTA per column: through DSMEM inside a thread-block cluster
//     of <= 16 CTAs (barrier.cluster per column) when the panel fits in the
//     cluster's shared memory, else through L2 with a cooperative grid barrier;
//     argmax pivot with first-index ties (np.argmax, dense.py:41), full-row swap,
//     scaling and rank-1 update exactly as dense.py:40-49;
//   * the panel kernel also emits the 32x32 unit-lower / upper diagonal-block
//     inverses (every triangular solve downstream is then a DMMA GEMM) and the
//     panel's interchanges as a (dst, src) row list, applied to all other
//     columns by one gather/scatter kernel (no per-swap serialisation);
//   * piv[k] = row swapped with k at step k (0-based) as lu_factor; an exactly
//     zero pivot reports column k (SingularMatrixError, dense.py:42-43);
//   * the composed row permutation perm (P B)[i] = B[perm[i]] is stored with the
//     factor so the solves apply all interchanges with one parallel gather.
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm.cuh"
#include "lu.cuh"
#include "panel.cuh"
#include "trsm.cuh"

namespace cg = cooperative_groups;

namespace fb {

namespace {

constexpr int PW = 32;         // sub-panel width (= diagonal block size of dinv)
constexpr int NB = 128;        // outer block (trailing-update K)
constexpr int LIST = 1 + 2 * 2 * PW;  // per-block swap list: cnt, dst[2PW], src[2PW]

// ---------------------------------------------------------------------------
// S = z B - A (B == nullptr: identity).  A/B real when their im pointer is null.
// ---------------------------------------------------------------------------
__global__ void shift_kernel(int n, double zr, double zi, const double* __restrict__ are,
                             const double* __restrict__ aim, long long lda,
                             const double* __restrict__ bre, const double* __restrict__ bim,
                             long long ldb, double* __restrict__ sre, double* __restrict__ sim,
                             long long lds) {
  long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / n), j = (int)(e % n);
    double ar = are[i * lda + j], ai = aim ? aim[i * lda + j] : 0.0;
    double br, bi;
    if (bre) {
      br = bre[i * ldb + j];
      bi = bim ? bim[i * ldb + j] : 0.0;
    } else {
      br = (i == j) ? 1.0 : 0.0;
      bi = 0.0;
    }
    // z*b (numpy complex product) then minus a (dense.py:101-103)
    double pr = __dsub_rn(__dmul_rn(zr, br), __dmul_rn(zi, bi));
    double pi = __dadd_rn(__dmul_rn(zr, bi), __dmul_rn(zi, br));
    sre[i * lds + j] = pr - ar;
    sim[i * lds + j] = pi - ai;
  }
}

// ---------------------------------------------------------------------------
// Row interchanges of one sub-panel, given as a (dst, src) list of <= 2*PW
// rows, applied to the columns [0, c0) u [c0+pw, n): stage the source rows of
// a 64-column strip in shared memory, then write them to their destinations.
// ---------------------------------------------------------------------------
constexpr int SW_COLS = 32;
__global__ void __launch_bounds__(256) swap_list_kernel(double* __restrict__ re, double* __restrict__ im,
                                                        long long ld, int ca, int cb, int cc, int cd,
                                                        const int* __restrict__ list) {
  __shared__ double sv[2 * PW][SW_COLS][2];
  __shared__ int sdst[2 * PW], ssrc[2 * PW];
  const int cnt = list[0];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    sdst[i] = list[1 + i];
    ssrc[i] = list[1 + 2 * PW + i];
  }
  __syncthreads();
  const int n1 = cb - ca, ncols = n1 + (cd - cc);
  const int j0 = blockIdx.x * SW_COLS;
  for (int e = threadIdx.x; e < cnt * SW_COLS; e += blockDim.x) {
    int i = e / SW_COLS, jj = e % SW_COLS, j = j0 + jj;
    if (j >= ncols) continue;
    int col = j < n1 ? ca + j : cc + (j - n1);
    long long o = (long long)ssrc[i] * ld + col;
    cp_async8(&sv[i][jj][0], re + o, true);
    cp_async8(&sv[i][jj][1], im + o, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int e = threadIdx.x; e < cnt * SW_COLS; e += blockDim.x) {
    int i = e / SW_COLS, jj = e % SW_COLS, j = j0 + jj;
    if (j >= ncols) continue;
    int col = j < n1 ? ca + j : cc + (j - n1);
    long long o = (long long)sdst[i] * ld + col;
    re[o] = sv[i][jj][0];
    im[o] = sv[i][jj][1];
  }
}

// ---------------------------------------------------------------------------
// Composed permutation from the per-block lists: idx starts as identity and
// each block maps idx'[dst] = idx[src] (one CTA, idx in shared memory).
// ---------------------------------------------------------------------------
__global__ void perm_kernel(int n, const int* __restrict__ lists, int* __restrict__ perm) {
  extern __shared__ int idx[];
  __shared__ int tmp[2 * PW];
  for (int i = threadIdx.x; i < n; i += blockDim.x) idx[i] = i;
  __syncthreads();
  const int nblk = ceil_div(n, PW);
  for (int b = 0; b < nblk; ++b) {
    const int* L = lists + (size_t)b * LIST;
    const int cnt = L[0];
    if (threadIdx.x < cnt) tmp[threadIdx.x] = idx[L[1 + 2 * PW + threadIdx.x]];
    __syncthreads();
    if (threadIdx.x < cnt) idx[L[1 + threadIdx.x]] = tmp[threadIdx.x];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = idx[i];
}

// out[i][j] = in[perm[i]][j] (gather = 1) or out[perm[i]][j] = in[i][j] (scatter)
__global__ void permute_rows_kernel(int n, int m, const int* __restrict__ perm, int gather,
                                    const double* __restrict__ ir, const double* __restrict__ ii,
                                    long long ldi, double* __restrict__ orr, double* __restrict__ oi,
                                    long long ldo) {
  long long total = (long long)n * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    int p = perm[i];
    if (gather) {
      orr[i * ldo + j] = ir[(long long)p * ldi + j];
      oi[i * ldo + j] = ii[(long long)p * ldi + j];
    } else {
      orr[(long long)p * ldo + j] = ir[i * ldi + j];
      oi[(long long)p * ldo + j] = ii[i * ldi + j];
    }
  }
}

}  // namespace

size_t zgetrf_scratch_bytes(int n) {
  (void)n;
  return panel_scratch_bytes();
}

// Factor side storage, in doubles: [nblk][4][PW][PW] diagonal inverses (L re/im,
// U re/im), then perm[n] ints, then nblk swap lists.
// ... then the per-block sweep operators G (trsm.cu) of the fused solves.
static size_t lists_doubles(int n) { return ((size_t)ceil_div(n, PW) * LIST + 1) / 2 + 2; }
size_t dinv_doubles(int n) {
  size_t nblk = ceil_div(n, PW);
  return nblk * 4 * PW * PW + ceil_div(n, 2) + lists_doubles(n) + gmat_doubles(n);
}
const int* factor_perm(const double* dinv, int n) {
  return reinterpret_cast<const int*>(dinv + (size_t)ceil_div(n, PW) * 4 * PW * PW);
}
static int* factor_lists(double* dinv, int n) {
  return reinterpret_cast<int*>(dinv + (size_t)ceil_div(n, PW) * 4 * PW * PW + ceil_div(n, 2));
}
const double* factor_gmat(const double* dinv, int n) {
  return dinv + (size_t)ceil_div(n, PW) * 4 * PW * PW + ceil_div(n, 2) + lists_doubles(n);
}

cudaError_t shift_launch(int n, double zr, double zi, const double* are, const double* aim,
                         long long lda, const double* bre, const double* bim, long long ldb,
                         double* sre, double* sim, long long lds, cudaStream_t st) {
  long long total = (long long)n * n;
  int blocks = (int)std::min<long long>((total + 255) / 256, 8 * kSMs);
  shift_kernel<<<blocks, 256, 0, st>>>(n, zr, zi, are, aim, lda, bre, bim, ldb, sre, sim, lds);
  count_launch();
  return cudaGetLastError();
}

cudaError_t permute_rows_launch(int n, int m, const int* perm, int gather, const double* ir,
                                const double* ii, long long ldi, double* orr, double* oi,
                                long long ldo, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  long long total = (long long)n * m;
  int blocks = (int)std::min<long long>((total + 255) / 256, 16 * kSMs);
  permute_rows_kernel<<<blocks, 256, 0, st>>>(n, m, perm, gather, ir, ii, ldi, orr, oi, ldo);
  count_launch();
  return cudaGetLastError();
}

// interchanges of one sub-panel on the columns [ca, cb) u [cc, cd)
static cudaError_t swap_list_launch(double* re, double* im, long long ld, int ca, int cb, int cc, int cd,
                                    const int* list, cudaStream_t st) {
  const int ncols = std::max(0, cb - ca) + std::max(0, cd - cc);
  if (ncols <= 0) return cudaSuccess;
  swap_list_kernel<<<ceil_div(ncols, SW_COLS), 256, 0, st>>>(re, im, ld, ca, std::max(ca, cb), cc,
                                                            std::max(cc, cd), list);
  count_launch();
  return cudaGetLastError();
}

// In-place LU of the planar n x n matrix (re, im, ld).  piv[n] (device, 0-based),
// info (device int, pre-set by caller to INT_MAX: stays INT_MAX on success,
// else 1 + first zero-pivot column), dinv = dinv_doubles(n) doubles.
//
// Look-ahead of depth one over two streams: the high-priority side stream P
// factors outer block k+1 (four panel launches + in-block updates) while the
// main stream S applies block k's bulk trailing update.  S finishes block k's
// next-block columns first and records F_k; P waits F_k, factors block k+1 and
// records E_{k+1}; S waits E_{k+1} before touching block k+1's results.  Row
// interchanges of block k outside the block (left L columns and the trailing
// matrix) are applied on S after its previous update, so P and S never write
// the same columns concurrently.
cudaError_t zgetrf(int n, double* re, double* im, long long ld, int* piv, int* info, double* dinv,
                   char* scratch, cudaStream_t st, const LuStreams* ls) {
  cudaError_t e;
  auto L = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW; };
  auto U = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW; };
  int* lists = factor_lists(dinv, n);
  const bool la = ls && ls->side && n > 2 * NB;
  cudaStream_t P = la ? ls->side : st;
  auto rec_wait = [&](cudaEvent_t ev, cudaStream_t from, cudaStream_t to) -> cudaError_t {
    if (from == to) return cudaSuccess;
    cudaError_t r = cudaEventRecord(ev, from);
    if (r) return r;
    return cudaStreamWaitEvent(to, ev, 0);
  };
  // factor outer block k on stream q (panels, in-block interchanges and updates)
  auto block_factor = [&](int k, cudaStream_t q) -> cudaError_t {
    const int nb = std::min(NB, n - k);
    cudaError_t r;
    for (int s = 0; s < nb; s += PW) {
      const int c0 = k + s, pw = std::min(PW, nb - s), blk = c0 / PW;
      int* list = lists + (size_t)blk * LIST;
      PanelArgs pa{};
      pa.re = re; pa.im = im; pa.ld = ld; pa.n = n; pa.c0 = c0; pa.pw = pw;
      pa.piv = piv; pa.info = info; pa.linv = L(blk); pa.uinv = U(blk); pa.list = list;
      if ((r = panel_launch(pa, scratch, q))) return r;
      if ((r = swap_list_launch(re, im, ld, k, c0, c0 + pw, k + nb, list, q))) return r;
      const int rest = k + nb - (c0 + pw);
      if (rest > 0) {
        double* br = re + (long long)c0 * ld + c0 + pw;
        double* bi = im + (long long)c0 * ld + c0 + pw;
        r = gemm(1, pw, rest, pw, op_n(L(blk), L(blk) + PW * PW, PW), op_n(br, bi, ld), br, bi, ld,
                 1.0, 0.0, 0.0, 0.0, q);
        if (r) return r;
        const int below = n - (c0 + pw);
        if (below > 0) {
          r = gemm(1, below, rest, pw,
                   op_n(re + (long long)(c0 + pw) * ld + c0, im + (long long)(c0 + pw) * ld + c0, ld),
                   op_n(br, bi, ld), re + (long long)(c0 + pw) * ld + c0 + pw,
                   im + (long long)(c0 + pw) * ld + c0 + pw, ld, -1.0, 0.0, 1.0, 0.0, q);
          if (r) return r;
        }
      }
    }
    return cudaSuccess;
  };
  // U12 = L11^{-1} A12 and A22 -= L21 U12 for the columns [c_lo, c_hi) of block k
  auto block_update = [&](int k, int c_lo, int c_hi, cudaStream_t q) -> cudaError_t {
    const int nb = std::min(NB, n - k);
    const int w = c_hi - c_lo;
    if (w <= 0) return cudaSuccess;
    cudaError_t r;
    for (int s = 0; s < nb; s += PW) {
      const int r0 = k + s, pw = std::min(PW, nb - s), blk = r0 / PW;
      double* xr = re + (long long)r0 * ld + c_lo;
      double* xi = im + (long long)r0 * ld + c_lo;
      r = gemm(1, pw, w, pw, op_n(L(blk), L(blk) + PW * PW, PW), op_n(xr, xi, ld), xr, xi, ld,
               1.0, 0.0, 0.0, 0.0, q);
      if (r) return r;
      const int rem = nb - s - pw;
      if (rem > 0) {
        r = gemm(1, rem, w, pw,
                 op_n(re + (long long)(r0 + pw) * ld + r0, im + (long long)(r0 + pw) * ld + r0, ld),
                 op_n(xr, xi, ld), re + (long long)(r0 + pw) * ld + c_lo,
                 im + (long long)(r0 + pw) * ld + c_lo, ld, -1.0, 0.0, 1.0, 0.0, q);
        if (r) return r;
      }
    }
    const int below = n - (k + nb);
    return gemm(1, below, w, nb,
                op_n(re + (long long)(k + nb) * ld + k, im + (long long)(k + nb) * ld + k, ld),
                op_n(re + (long long)k * ld + c_lo, im + (long long)k * ld + c_lo, ld),
                re + (long long)(k + nb) * ld + c_lo, im + (long long)(k + nb) * ld + c_lo, ld, -1.0, 0.0,
                1.0, 0.0, q);
  };

  if (la && (e = rec_wait(ls->ev_s, st, P))) return e;  // P sees the shifted matrix
  if ((e = block_factor(0, P))) return e;
  for (int k = 0; k < n; k += NB) {
    const int nb = std::min(NB, n - k);
    if (la && (e = rec_wait(ls->ev_p, P, st))) return e;  // E_k: block k factored
    // block k's interchanges outside the block (left L columns, trailing matrix)
    for (int s = 0; s < nb; s += PW) {
      const int c0 = k + s, pw = std::min(PW, nb - s);
      (void)pw;
      const int* list = lists + (size_t)(c0 / PW) * LIST;
      if ((e = swap_list_launch(re, im, ld, 0, k, k + nb, n, list, st))) return e;
    }
    if (k + nb >= n) break;
    const int next_hi = std::min(n, k + 2 * NB);
    if ((e = block_update(k, k + nb, next_hi, st))) return e;  // next block's columns first
    if (la) {
      if ((e = rec_wait(ls->ev_s, st, P))) return e;  // F_k
      if ((e = block_factor(k + nb, P))) return e;
      if ((e = block_update(k, next_hi, n, st))) return e;  // bulk, overlapped with the panel
    } else {
      if ((e = block_update(k, next_hi, n, st))) return e;
      if ((e = block_factor(k + nb, st))) return e;
    }
  }
  // composed permutation for the solves
  size_t psmem = sizeof(int) * (size_t)n;
  static bool pcfg = false;
  if (!pcfg) {
    cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    pcfg = true;
  }
  if (psmem > 200 * 1024) return cudaErrorInvalidValue;
  perm_kernel<<<1, 256, psmem, st>>>(n, lists, const_cast<int*>(factor_perm(dinv, n)));
  count_launch();
  if ((e = cudaGetLastError())) return e;
  return gmat_launch(n, re, im, ld, dinv, const_cast<double*>(factor_gmat(dinv, n)), st);
}

// Solve op(A) X = B in place for X (n x nrhs planar, ldx) from zgetrf output.
// adjoint = 0: A X = B (dense.py:62-74); adjoint = 1: A^H X = B (dense.py:75-87).
// tmp: n*nrhs*2 doubles of scratch for the row permutation.
cudaError_t zgetrs(int n, int nrhs, const double* re, const double* im, long long ld, const int* piv,
                   const double* dinv, int adjoint, double* xr, double* xi, long long ldx, double* tmp,
                   cudaStream_t st) {
  cudaError_t e;
  (void)piv;
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int nblk = ceil_div(n, PW);
  const int* perm = factor_perm(dinv, n);
  double* tr = tmp;
  double* ti = tmp + (size_t)n * nrhs;
  auto L = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW; };
  auto U = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW; };
  auto row = [&](const double* p, int r, int c) { return p + (long long)r * ld + c; };
  static const bool blocked = getenv("FB_SOLVE_BLOCKED") != nullptr;  // A/B switch for tests
  if (!blocked) {
    const double* gm = factor_gmat(dinv, n);
    if (!adjoint) {
      if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
      if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
      if ((e = permute_rows_launch(n, nrhs, perm, 1, tr, ti, nrhs, xr, xi, ldx, st))) return e;
      if ((e = sweep_launch(0, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st))) return e;
      return sweep_launch(1, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st);
    }
    if ((e = sweep_launch(2, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st))) return e;
    if ((e = sweep_launch(3, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st))) return e;
    if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    return permute_rows_launch(n, nrhs, perm, 0, tr, ti, nrhs, xr, xi, ldx, st);
  }
  if (!adjoint) {
    // X <- P X (one gather through the scratch copy)
    if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = permute_rows_launch(n, nrhs, perm, 1, tr, ti, nrhs, xr, xi, ldx, st))) return e;
    for (int b = 0; b < nblk; ++b) {  // forward, unit L
      const int r0 = b * PW, pw = std::min(PW, n - r0);
      double* x0r = xr + (long long)r0 * ldx;
      double* x0i = xi + (long long)r0 * ldx;
      if ((e = gemm(1, pw, nrhs, pw, op_n(L(b), L(b) + PW * PW, PW), op_n(x0r, x0i, ldx), x0r, x0i,
                    ldx, 1.0, 0.0, 0.0, 0.0, st)))
        return e;
      const int below = n - r0 - pw;
      if (below > 0 &&
          (e = gemm(1, below, nrhs, pw, op_n(row(re, r0 + pw, r0), row(im, r0 + pw, r0), ld),
                    op_n(x0r, x0i, ldx), xr + (long long)(r0 + pw) * ldx,
                    xi + (long long)(r0 + pw) * ldx, ldx, -1.0, 0.0, 1.0, 0.0, st)))
        return e;
    }
    for (int b = nblk - 1; b >= 0; --b) {  // backward, U
      const int r0 = b * PW, pw = std::min(PW, n - r0);
      double* x0r = xr + (long long)r0 * ldx;
      double* x0i = xi + (long long)r0 * ldx;
      if ((e = gemm(1, pw, nrhs, pw, op_n(U(b), U(b) + PW * PW, PW), op_n(x0r, x0i, ldx), x0r, x0i,
                    ldx, 1.0, 0.0, 0.0, 0.0, st)))
        return e;
      if (r0 > 0 && (e = gemm(1, r0, nrhs, pw, op_n(row(re, 0, r0), row(im, 0, r0), ld),
                              op_n(x0r, x0i, ldx), xr, xi, ldx, -1.0, 0.0, 1.0, 0.0, st)))
        return e;
    }
    return cudaSuccess;
  }
  // A^H = U^H L^H P: forward with U^H, backward with L^H, then X <- P^T X
  for (int b = 0; b < nblk; ++b) {
    const int r0 = b * PW, pw = std::min(PW, n - r0);
    double* x0r = xr + (long long)r0 * ldx;
    double* x0i = xi + (long long)r0 * ldx;
    if ((e = gemm(1, pw, nrhs, pw, op_c(U(b), U(b) + PW * PW, PW), op_n(x0r, x0i, ldx), x0r, x0i, ldx,
                  1.0, 0.0, 0.0, 0.0, st)))
      return e;
    const int below = n - r0 - pw;
    if (below > 0 &&
        (e = gemm(1, below, nrhs, pw, op_c(row(re, r0, r0 + pw), row(im, r0, r0 + pw), ld),
                  op_n(x0r, x0i, ldx), xr + (long long)(r0 + pw) * ldx, xi + (long long)(r0 + pw) * ldx,
                  ldx, -1.0, 0.0, 1.0, 0.0, st)))
      return e;
  }
  for (int b = nblk - 1; b >= 0; --b) {
    const int r0 = b * PW, pw = std::min(PW, n - r0);
    double* x0r = xr + (long long)r0 * ldx;
    double* x0i = xi + (long long)r0 * ldx;
    if ((e = gemm(1, pw, nrhs, pw, op_c(L(b), L(b) + PW * PW, PW), op_n(x0r, x0i, ldx), x0r, x0i, ldx,
                  1.0, 0.0, 0.0, 0.0, st)))
      return e;
    if (r0 > 0 && (e = gemm(1, r0, nrhs, pw, op_c(row(re, r0, 0), row(im, r0, 0), ld),
                            op_n(x0r, x0i, ldx), xr, xi, ldx, -1.0, 0.0, 1.0, 0.0, st)))
      return e;
  }
  if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
  return permute_rows_launch(n, nrhs, perm, 0, tr, ti, nrhs, xr, xi, ldx, st);
}

}  // namespace fb
