// Dense shifted complex LU with partial pivoting and its multi-RHS solves,
// batched over contour points.
//
// Restates feastlib's dense backend (dense.py:30-88, _DenseOps dense.py:91-117)
// as a blocked algorithm for sm_100a:
//   * shift formation S_e = z_e B - A (dense.py:97-103), planar complex;
//   * right-looking blocked LU, outer block NB = 256 (trailing update is one
//     DMMA ZGEMM with K = 256), inner sub-panels of PW = 32 columns factored by
//     panel.cu (cluster/DSMEM exchange, one pivot per column);
//   * the panel kernel also emits the 32x32 unit-lower diagonal-block inverse
//     (the in-factorization U12 = L11^-1 A12 is then a DMMA GEMM) and the
//     panel's interchanges as a (dst, src) row list, applied to the other
//     columns by one gather/scatter kernel;
//   * piv[k] = row swapped with k at step k (0-based) as lu_factor; an exactly
//     zero pivot reports column k (SingularMatrixError, dense.py:42-43);
//   * the composed row permutation perm, (P B)[i] = B[perm[i]], is stored with
//     the factor so the solves apply all interchanges with one gather.
//
// Every routine takes a strided BATCH of independent factorizations (the
// Ne shifts of one contour pass): one launch per step covers all of them, so
// the latency-bound panel steps of different shifts run side by side on
// different SMs and the trailing GEMMs get Ne times more tiles.  This is the
// GPU form of the reference's contour-parallel pre-factorization
// (_driver.py:46-54): each factorization is computed exactly as it would be
// alone, so results do not depend on the batch composition.
#include <cstdlib>
#include <utility>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"
#include "lu.cuh"
#include "panel.cuh"
#include "trsm.cuh"

namespace fb {

namespace {

constexpr int PW = 32;                 // sub-panel width (= diagonal block size of dinv)
// outer block (trailing-update K): 256 is +3 % over 128 at N = 4096 and 8192 (profiles/r01_lu_nb_rpc_sweep.txt)
static int outer_nb() { return 256; }
constexpr int LIST = 1 + 2 * 2 * PW;   // per-block swap list: cnt, dst[2PW], src[2PW]

// S_b = z_b B - A (B == nullptr: identity); item b = blockIdx.y.
struct ShiftZ {
  double zr[kMaxBatch], zi[kMaxBatch];
};
__global__ void shift_kernel(int n, ShiftZ z, const double* __restrict__ are, const double* __restrict__ aim,
                             long long lda, const double* __restrict__ bre, const double* __restrict__ bim,
                             long long ldb, double* __restrict__ sre, double* __restrict__ sim, long long lds,
                             long long ss) {
  const int b = blockIdx.y;
  const double zr = z.zr[b], zi = z.zi[b];
  sre += b * ss;
  sim += b * ss;
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

// Row interchanges of one sub-panel, given as a (dst, src) list of <= 2*PW
// rows, applied to the columns [ca, cb) u [cc, cd): stage the source rows of a
// 32-column strip in shared memory (cp.async), then write them to their
// destinations.  Item b = blockIdx.y.
constexpr int SW_COLS = 32;
__global__ void __launch_bounds__(256) swap_list_kernel(double* __restrict__ re, double* __restrict__ im,
                                                        long long ld, long long slu, int ca, int cb, int cc,
                                                        int cd, const int* __restrict__ list,
                                                        long long slist) {
  __shared__ double sv[2 * PW][SW_COLS][2];
  __shared__ int sdst[2 * PW], ssrc[2 * PW];
  const int b = blockIdx.y;
  re += b * slu;
  im += b * slu;
  list += b * slist;
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

// Composed permutation from the per-block lists: idx starts as identity and
// each block maps idx'[dst] = idx[src] (one CTA per item, idx in smem).
__global__ void perm_kernel(int n, const int* __restrict__ lists, int* __restrict__ perm, long long sint) {
  extern __shared__ int idx[];
  __shared__ int tmp[2 * PW];
  lists += blockIdx.x * sint;
  perm += blockIdx.x * sint;
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

// out_b[i][j] = in_b[perm_b[i]][j] (gather) or out_b[perm_b[i]][j] = in_b[i][j]
// (scatter); item b = blockIdx.y, strides may be 0 for a shared input.
__global__ void permute_rows_kernel(int n, int m, const int* __restrict__ perm, long long sperm, int gather,
                                    const double* __restrict__ ir, const double* __restrict__ ii,
                                    long long ldi, long long sin_, double* __restrict__ orr,
                                    double* __restrict__ oi, long long ldo, long long sout) {
  const int b = blockIdx.y;
  perm += b * sperm;
  ir += b * sin_;
  ii += b * sin_;
  orr += b * sout;
  oi += b * sout;
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

__global__ void fill_int_kernel(int* p, int v, int count) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) p[i] = v;
}

}  // namespace

// FB_PANEL_EVENTS (debug): CUDA events around every panel launch
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_pev;
static bool panel_events_on() {
  static const bool on = getenv("FB_PANEL_EVENTS") != nullptr;
  return on;
}
static void panel_events_push(cudaEvent_t a, cudaEvent_t b) { g_pev.emplace_back(a, b); }
double panel_events_read_ms(int* count) {
  double tot = 0.0;
  for (auto& p : g_pev) {
    cudaEventSynchronize(p.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.first, p.second);
    tot += ms;
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  *count = (int)g_pev.size();
  g_pev.clear();
  return tot;
}

size_t zgetrf_scratch_bytes(int n, int count) {
  (void)n;
  return panel_scratch_bytes() * (size_t)count;
}

// Factor side storage, in doubles: [nblk][4][PW][PW] (the unit-lower diagonal
// inverses L re/im used by the factorization; the second half is unused), then
// perm[n] ints, then nblk swap lists, then the per-block substitution operators
// (trsm.cu tdiag_kernel) of the fused solves.
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

cudaError_t shift_launch(int n, int count, const double* zr, const double* zi, const double* are,
                         const double* aim, long long lda, const double* bre, const double* bim,
                         long long ldb, double* sre, double* sim, long long lds, long long ss, cudaStream_t st) {
  if (n <= 0 || count <= 0) return cudaSuccess;
  if (count > kMaxBatch) return cudaErrorInvalidValue;
  ShiftZ z{};
  for (int b = 0; b < count; ++b) {
    z.zr[b] = zr[b];
    z.zi[b] = zi[b];
  }
  long long total = (long long)n * n;
  int blocks = (int)std::min<long long>((total + 255) / 256, std::max(1, 8 * kSMs / count));
  shift_kernel<<<dim3(blocks, count), 256, 0, st>>>(n, z, are, aim, lda, bre, bim, ldb, sre, sim, lds, ss);
  count_launch();
  return cudaGetLastError();
}

cudaError_t permute_rows_launch(int n, int m, int count, const int* perm, long long sperm, int gather,
                                const double* ir, const double* ii, long long ldi, long long sin_, double* orr,
                                double* oi, long long ldo, long long sout, cudaStream_t st) {
  if (n <= 0 || m <= 0 || count <= 0) return cudaSuccess;
  long long total = (long long)n * m;
  int blocks = (int)std::min<long long>((total + 255) / 256, std::max(1, 16 * kSMs / count));
  permute_rows_kernel<<<dim3(blocks, count), 256, 0, st>>>(n, m, perm, sperm, gather, ir, ii, ldi, sin_, orr,
                                                            oi, ldo, sout);
  count_launch();
  return cudaGetLastError();
}

// interchanges of one sub-panel on the columns [ca, cb) u [cc, cd), all items
static cudaError_t swap_list_launch(const LuBatch& f, int ca, int cb, int cc, int cd, const int* list,
                                    cudaStream_t st) {
  const int ncols = std::max(0, cb - ca) + std::max(0, cd - cc);
  if (ncols <= 0) return cudaSuccess;
  swap_list_kernel<<<dim3(ceil_div(ncols, SW_COLS), f.count), 256, 0, st>>>(
      f.re, f.im, f.ld, f.slu, ca, std::max(ca, cb), cc, std::max(cc, cd), list, 2 * f.sdinv);
  count_launch();
  return cudaGetLastError();
}

// In-place LU of a strided batch of planar n x n matrices.  piv (0-based),
// info[b] = INT_MAX on success else 1 + first zero-pivot column (set here),
// dinv = dinv_doubles(n) doubles per item.
//
// Look-ahead of depth one over two streams: the high-priority side stream P
// factors outer block k+1 (four panel launches + in-block updates) while the
// main stream S applies block k's bulk trailing update.  S finishes block k's
// next-block columns first and records F_k; P waits F_k, factors block k+1 and
// records E_{k+1}; S waits E_{k+1} before touching block k+1's results.  Row
// interchanges of block k outside the block (left L columns and the trailing
// matrix) are applied on S after its previous update, so P and S never write
// the same columns concurrently.
cudaError_t zgetrf_batched(int n, const LuBatch& f, char* scratch, cudaStream_t st, const LuStreams* ls) {
  cudaError_t e;
  if (n <= 0 || f.count <= 0) return cudaSuccess;
  const int NB = outer_nb();
  const int B = f.count;
  const long long ld = f.ld, slu = f.slu, sd = f.sdinv;
  double* re = f.re;
  double* im = f.im;
  auto L = [&](int blk) { return f.dinv + (size_t)blk * 4 * PW * PW; };
  auto U = [&](int blk) { return f.dinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW; };
  int* lists = factor_lists(f.dinv, n);
  const bool la = ls && ls->side && n > 2 * NB;
  cudaStream_t P = la ? ls->side : st;
  auto rec_wait = [&](cudaEvent_t ev, cudaStream_t from, cudaStream_t to) -> cudaError_t {
    if (from == to) return cudaSuccess;
    cudaError_t r = cudaEventRecord(ev, from);
    if (r) return r;
    return cudaStreamWaitEvent(to, ev, 0);
  };
  fill_int_kernel<<<ceil_div(B, 128), 128, 0, st>>>(f.info, 0x7fffffff, B);
  count_launch();
  // tensor maps over the batch of factor matrices: the bulk trailing updates are TMA-fed (gemm_tma.cu)
  LuTmaMaps tma;
  lu_tma_maps_make(&tma, re, im, n, ld, slu, B);
  // factor outer block k on stream q (panels, in-block interchanges and updates)
  auto block_factor = [&](int k, cudaStream_t q) -> cudaError_t {
    const int nb = std::min(NB, n - k);
    cudaError_t r;
    for (int s = 0; s < nb; s += PW) {
      const int c0 = k + s, pw = std::min(PW, nb - s), blk = c0 / PW;
      int* list = lists + (size_t)blk * LIST;
      PanelArgs pa{};
      pa.re = re; pa.im = im; pa.ld = ld; pa.n = n; pa.c0 = c0; pa.pw = pw;
      pa.piv = f.piv; pa.info = f.info; pa.linv = L(blk); pa.uinv = U(blk); pa.list = list;
      pa.slu = slu; pa.spiv = f.spiv; pa.sdinv = sd;
      if (panel_events_on()) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, q);
        if ((r = panel_launch(pa, B, scratch, q))) return r;
        cudaEventRecord(e1, q);
        panel_events_push(e0, e1);
      } else if ((r = panel_launch(pa, B, scratch, q))) {
        return r;
      }
      if ((r = swap_list_launch(f, k, c0, c0 + pw, k + nb, list, q))) return r;
      const int rest = k + nb - (c0 + pw);
      if (rest > 0) {
        double* br = re + (long long)c0 * ld + c0 + pw;
        double* bi = im + (long long)c0 * ld + c0 + pw;
        r = gemm(1, pw, rest, pw, op_n(L(blk), L(blk) + PW * PW, PW), op_n(br, bi, ld), br, bi, ld, 1.0, 0.0,
                 0.0, 0.0, q, nullptr, 1, B, sd, slu, slu);
        if (r) return r;
        const int below = n - (c0 + pw);
        if (below > 0) {
          r = gemm(1, below, rest, pw,
                   op_n(re + (long long)(c0 + pw) * ld + c0, im + (long long)(c0 + pw) * ld + c0, ld),
                   op_n(br, bi, ld), re + (long long)(c0 + pw) * ld + c0 + pw,
                   im + (long long)(c0 + pw) * ld + c0 + pw, ld, -1.0, 0.0, 1.0, 0.0, q, nullptr, 1, B, slu,
                   slu, slu);
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
      r = gemm(1, pw, w, pw, op_n(L(blk), L(blk) + PW * PW, PW), op_n(xr, xi, ld), xr, xi, ld, 1.0, 0.0, 0.0,
               0.0, q, nullptr, 1, B, sd, slu, slu);
      if (r) return r;
      const int rem = nb - s - pw;
      if (rem > 0) {
        r = gemm(1, rem, w, pw,
                 op_n(re + (long long)(r0 + pw) * ld + r0, im + (long long)(r0 + pw) * ld + r0, ld),
                 op_n(xr, xi, ld), re + (long long)(r0 + pw) * ld + c_lo, im + (long long)(r0 + pw) * ld + c_lo,
                 ld, -1.0, 0.0, 1.0, 0.0, q, nullptr, 1, B, slu, slu, slu);
        if (r) return r;
      }
    }
    const int below = n - (k + nb);
    if (tma.ok && nb % 16 == 0 && (c_lo & 1) == 0 && below >= 64)
      return lu_trailing_tma(tma, re, im, ld, slu, B, below, w, nb, k + nb, k, k, c_lo, k + nb, c_lo, q);
    return gemm(1, below, w, nb, op_n(re + (long long)(k + nb) * ld + k, im + (long long)(k + nb) * ld + k, ld),
                op_n(re + (long long)k * ld + c_lo, im + (long long)k * ld + c_lo, ld),
                re + (long long)(k + nb) * ld + c_lo, im + (long long)(k + nb) * ld + c_lo, ld, -1.0, 0.0, 1.0,
                0.0, q, nullptr, 1, B, slu, slu, slu);
  };

  if (la && (e = rec_wait(ls->ev_s, st, P))) return e;  // P sees the shifted matrices
  if ((e = block_factor(0, P))) return e;
  for (int k = 0; k < n; k += NB) {
    const int nb = std::min(NB, n - k);
    if (la && (e = rec_wait(ls->ev_p, P, st))) return e;  // E_k: block k factored
    // block k's interchanges outside the block (left L columns, trailing matrix)
    for (int s = 0; s < nb; s += PW) {
      const int* list = lists + (size_t)((k + s) / PW) * LIST;
      if ((e = swap_list_launch(f, 0, k, k + nb, n, list, st))) return e;
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
  // composed permutation and the sweeps' diagonal-block operators for the solves
  size_t psmem = sizeof(int) * (size_t)n;
  static DevOnce pcfg;
  if (pcfg.first()) cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (psmem > 200 * 1024) return cudaErrorInvalidValue;
  perm_kernel<<<B, 256, psmem, st>>>(n, lists, const_cast<int*>(factor_perm(f.dinv, n)), 2 * sd);
  count_launch();
  if ((e = cudaGetLastError())) return e;
  return gmat_launch(n, B, re, im, ld, slu, f.dinv, sd, const_cast<double*>(factor_gmat(f.dinv, n)), st);
}

// Solve op(A_b) X_b = B_b for a batch: item b reads its right-hand sides from
// rhs + b*srhs (srhs = 0: one shared block, e.g. the contour pass's Y) and
// writes X_b = x + b*sx.  adjoint = 0: A X = B (dense.py:62-74); adjoint = 1:
// A^H X = B (dense.py:75-87).  tmp: count*n*nrhs*2 doubles (adjoint only).
cudaError_t zgetrs_batched(int n, int nrhs, const LuBatch& f, int adjoint, const double* rr, const double* ri,
                           long long ldr, long long srhs, double* xr, double* xi, long long ldx, long long sx,
                           double* tmp, cudaStream_t st) {
  cudaError_t e;
  if (n <= 0 || nrhs <= 0 || f.count <= 0) return cudaSuccess;
  const int B = f.count;
  const int* perm = factor_perm(f.dinv, n);
  const double* gm = factor_gmat(f.dinv, n);
  if (!adjoint) {
    // X_b <- P_b B_b (one gather), then the L and U sweeps
    if ((e = permute_rows_launch(n, nrhs, B, perm, 2 * f.sdinv, 1, rr, ri, ldr, srhs, xr, xi, ldx, sx, st)))
      return e;
    if ((e = sweep_launch(0, n, nrhs, B, f.re, f.im, f.ld, f.slu, f.dinv, gm, f.sdinv, xr, xi, ldx, sx, st)))
      return e;
    return sweep_launch(1, n, nrhs, B, f.re, f.im, f.ld, f.slu, f.dinv, gm, f.sdinv, xr, xi, ldx, sx, st);
  }
  // A^H = U^H L^H P: U^H and L^H sweeps on a copy, then X_b <- P_b^T (scatter).
  // The copy's leading dimension is even so the sweeps take the 16-byte path
  // even when M0 has shrunk to an odd column count.
  const int tld = zgetrs_tmp_ld(nrhs);
  const long long st_ = (long long)n * tld;
  double* tr = tmp;
  double* ti = tmp + (size_t)B * st_;
  for (int b = 0; b < B; ++b) {
    if ((e = cudaMemcpy2DAsync(tr + b * st_, tld * 8, rr + b * srhs, ldr * 8, nrhs * 8, n,
                               cudaMemcpyDeviceToDevice, st)))
      return e;
    if ((e = cudaMemcpy2DAsync(ti + b * st_, tld * 8, ri + b * srhs, ldr * 8, nrhs * 8, n,
                               cudaMemcpyDeviceToDevice, st)))
      return e;
  }
  if ((e = sweep_launch(2, n, nrhs, B, f.re, f.im, f.ld, f.slu, f.dinv, gm, f.sdinv, tr, ti, tld, st_, st)))
    return e;
  if ((e = sweep_launch(3, n, nrhs, B, f.re, f.im, f.ld, f.slu, f.dinv, gm, f.sdinv, tr, ti, tld, st_, st)))
    return e;
  return permute_rows_launch(n, nrhs, B, perm, 2 * f.sdinv, 0, tr, ti, tld, st_, xr, xi, ldx, sx, st);
}

}  // namespace fb
