// extern "C" boundary of libfeastb200.so (declared in include/feast_b200.h).
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../../include/feast_b200.h"
#include "band.cuh"
#include "common.cuh"
#include "csr.cuh"
#include "gemm.cuh"
#include "lu.cuh"
#include "misc.cuh"

namespace fb {
void panel_profile_read(unsigned long long* out);
void panel_wall_read(unsigned long long* out4);
double panel_events_read_ms(int* count);
void reduced_profile_read(unsigned long long* out);
void reduced_cluster_profile_read(unsigned long long* out);
}

std::atomic<long long> fb::g_launches{0};

struct fb_ctx : fb::Ctx {
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int* dev_word = nullptr;   // small device scratch for status words
  int* host_word = nullptr;  // pinned mirror
  long long launches = 0;
  fb::LuStreams lu{};        // look-ahead side stream + events of zgetrf
};

using fb::FB_ERR_ALLOC;
using fb::FB_ERR_ARG;
using fb::FB_ERR_CUDA;
using fb::FB_ERR_SINGULAR;
using fb::FB_OK;

namespace {

int set_err(fb_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FB_OK;
  if (c) snprintf(c->err, sizeof(c->err), "%s: %s", what, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? FB_ERR_ALLOC : FB_ERR_CUDA;
}

int ensure_scratch(fb_ctx* c, size_t bytes) {
  if (bytes <= c->scratch_bytes) return FB_OK;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_err(c, e, "sync before scratch growth");
  if (c->scratch) cudaFree(c->scratch);
  c->scratch = nullptr;
  c->scratch_bytes = 0;
  size_t want = bytes + bytes / 4 + (1 << 20);
  e = cudaMalloc(&c->scratch, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(c, e, "scratch cudaMalloc");
  }
  c->scratch_bytes = want;
  return FB_OK;
}

int use_device(fb_ctx* c) {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != c->device) {
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return set_err(c, e, "cudaSetDevice");
  }
  return FB_OK;
}

#define CTX_GUARD(c)                  \
  do {                                \
    if (!(c)) return FB_ERR_ARG;      \
    int _g = use_device(c);           \
    if (_g) return _g;                \
  } while (0)

fb::Opnd make_op(char op, const double* re, const double* im, int64_t ld) {
  switch (op) {
    case 'T': case 't': return fb::op_t(re, im, ld);
    case 'C': case 'c': return fb::op_c(re, im, ld);
    default: return fb::op_n(re, im, ld);
  }
}

}  // namespace

extern "C" {

int fb_abi_version(void) { return FB_ABI_VERSION; }

int fb_ctx_create(int device, void* stream, fb_ctx** out) {
  if (!out) return FB_ERR_ARG;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? FB_ERR_ALLOC : FB_ERR_CUDA;
  fb_ctx* c = new fb_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  c->err[0] = 0;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  e = cudaMalloc(&c->dev_word, 64 * sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&c->host_word, 64 * sizeof(int));
  if (e != cudaSuccess) {
    delete c;
    return FB_ERR_ALLOC;
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&c->lu.side, cudaStreamNonBlocking, hi) == cudaSuccess) {
    cudaEventCreateWithFlags(&c->lu.ev_s, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->lu.ev_p, cudaEventDisableTiming);
  } else {
    c->lu.side = nullptr;
    cudaGetLastError();
  }
  *out = c;
  return FB_OK;
}

int fb_ctx_destroy(fb_ctx* c) {
  if (!c) return FB_OK;
  use_device(c);
  cudaStreamSynchronize(c->stream);
  if (c->lu.side) {
    cudaStreamSynchronize(c->lu.side);
    cudaEventDestroy(c->lu.ev_s);
    cudaEventDestroy(c->lu.ev_p);
    cudaStreamDestroy(c->lu.side);
  }
  if (c->scratch) cudaFree(c->scratch);
  if (c->dev_word) cudaFree(c->dev_word);
  if (c->host_word) cudaFreeHost(c->host_word);
  delete c;
  return FB_OK;
}

int fb_ctx_set_stream(fb_ctx* c, void* stream) {
  if (!c) return FB_ERR_ARG;
  c->stream = static_cast<cudaStream_t>(stream);
  return FB_OK;
}

int fb_ctx_synchronize(fb_ctx* c) {
  CTX_GUARD(c);
  return set_err(c, cudaStreamSynchronize(c->stream), "synchronize");
}

const char* fb_ctx_last_error(const fb_ctx* c) { return c ? c->err : "null context"; }

int64_t fb_ctx_launch_count(const fb_ctx* c) {
  (void)c;
  return fb::g_launches.load(std::memory_order_relaxed);
}

int fb_dense_shift(fb_ctx* c, int n, double zr, double zi, const double* are, const double* aim,
                   int64_t lda, const double* bre, const double* bim, int64_t ldb, double* sre,
                   double* sim, int64_t lds) {
  return fb_dense_shift_batched(c, 1, n, &zr, &zi, are, aim, lda, bre, bim, ldb, sre, sim, lds, 0);
}

int fb_dense_shift_batched(fb_ctx* c, int count, int n, const double* zr, const double* zi, const double* are,
                           const double* aim, int64_t lda, const double* bre, const double* bim, int64_t ldb,
                           double* sre, double* sim, int64_t lds, int64_t s_stride) {
  CTX_GUARD(c);
  if (n < 0 || count < 0 || count > fb::kMaxBatch || !are || !sre || !sim || !zr || !zi) return FB_ERR_ARG;
  return set_err(c, fb::shift_launch(n, count, zr, zi, are, aim, lda, bre, bim, ldb, sre, sim, lds, s_stride,
                                     c->stream),
                 "dense_shift");
}

size_t fb_zgetrf_dinv_doubles(int n) { return fb::dinv_doubles(n); }

int fb_zgetrf(fb_ctx* c, int n, double* re, double* im, int64_t ld, int* piv, double* dinv, int* info) {
  return fb_zgetrf_batched(c, 1, n, re, im, ld, 0, piv, 0, dinv, 0, info);
}

int fb_zgetrf_batched(fb_ctx* c, int count, int n, double* re, double* im, int64_t ld, int64_t lu_stride,
                      int* piv, int64_t piv_stride, double* dinv, int64_t dinv_stride, int* info) {
  CTX_GUARD(c);
  if (n < 0 || count < 0 || !re || !im || !piv || !dinv || !info) return FB_ERR_ARG;
  if (count == 0 || n == 0) return FB_OK;
  int r = ensure_scratch(c, fb::zgetrf_scratch_bytes(n, count));
  if (r) return r;
  fb::LuBatch f{count, re, im, ld, lu_stride, piv, piv_stride, info, dinv, dinv_stride};
  return set_err(c, fb::zgetrf_batched(n, f, (char*)c->scratch, c->stream, &c->lu), "zgetrf");
}

int fb_read_info(fb_ctx* c, const int* info, int* bad_col) {
  return fb_read_info_batched(c, 1, info, bad_col);
}

int fb_read_info_batched(fb_ctx* c, int count, const int* info, int* bad_cols) {
  CTX_GUARD(c);
  if (count < 0 || count > 64) return FB_ERR_ARG;
  cudaError_t e = cudaMemcpyAsync(c->host_word, info, sizeof(int) * count, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_err(c, e, "read_info");
  int rc = FB_OK;
  for (int b = 0; b < count; ++b) {
    int v = c->host_word[b];
    if (bad_cols) bad_cols[b] = (v == INT_MAX) ? -1 : v - 1;
    if (v != INT_MAX) rc = FB_ERR_SINGULAR;
  }
  return rc;
}

int fb_zgetrs(fb_ctx* c, int n, int nrhs, const double* re, const double* im, int64_t ld, const int* piv,
              const double* dinv, int adjoint, double* xr, double* xi, int64_t ldx) {
  CTX_GUARD(c);
  if (n < 0 || nrhs < 0 || !xr || !xi) return FB_ERR_ARG;
  if (n == 0 || nrhs == 0) return FB_OK;
  // in place: the right-hand sides go through the scratch first
  const int tld = fb::zgetrs_tmp_ld(nrhs);
  const size_t plane = (size_t)n * (size_t)tld;
  int r = ensure_scratch(c, sizeof(double) * 4 * plane);
  if (r) return r;
  double* tr = (double*)c->scratch;
  double* ti = tr + plane;
  cudaError_t e = cudaMemcpy2DAsync(tr, tld * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(ti, tld * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, c->stream);
  if (e != cudaSuccess) return set_err(c, e, "zgetrs copy");
  fb::LuBatch f{1, const_cast<double*>(re), const_cast<double*>(im), ld, 0, const_cast<int*>(piv), 0,
                nullptr, const_cast<double*>(dinv), 0};
  return set_err(c, fb::zgetrs_batched(n, nrhs, f, adjoint, tr, ti, tld, 0, xr, xi, ldx, 0, tr + 2 * plane,
                                       c->stream),
                 "zgetrs");
}

int fb_zgetrs_batched(fb_ctx* c, int count, int n, int nrhs, const double* re, const double* im, int64_t ld,
                      int64_t lu_stride, const int* piv, int64_t piv_stride, const double* dinv,
                      int64_t dinv_stride, int adjoint, const double* br, const double* bi, int64_t ldb,
                      int64_t b_stride, double* xr, double* xi, int64_t ldx, int64_t x_stride) {
  CTX_GUARD(c);
  if (n < 0 || nrhs < 0 || count < 0 || !xr || !xi || !br || !bi) return FB_ERR_ARG;
  if (n == 0 || nrhs == 0 || count == 0) return FB_OK;
  int r = ensure_scratch(c, sizeof(double) * 2 * (size_t)count * n * fb::zgetrs_tmp_ld(nrhs));
  if (r) return r;
  fb::LuBatch f{count, const_cast<double*>(re), const_cast<double*>(im), ld, lu_stride, const_cast<int*>(piv),
                piv_stride, nullptr, const_cast<double*>(dinv), dinv_stride};
  return set_err(c, fb::zgetrs_batched(n, nrhs, f, adjoint, br, bi, ldb, b_stride, xr, xi, ldx, x_stride,
                                       (double*)c->scratch, c->stream),
                 "zgetrs");
}

int fb_splitmix(fb_ctx* c, uint64_t seed, int64_t off_re, int64_t off_im, int n, int m, double* re,
                double* im, int64_t ld) {
  CTX_GUARD(c);
  return set_err(c, fb::splitmix_launch(seed, off_re, off_im, n, m, re, im, ld, c->stream), "splitmix");
}

// Coefficients evaluated as numpy does (kernel.py:117-123):
//   sym : (w/2.0) * (r*exp(i theta) * x).real
//   herm: ((w/4.0) * r) * exp(+-i theta), then times x
static void acc_coeffs(int variant, double w, double r, double theta, int* mode, double* h, double* cr,
                       double* ci) {
  double cth = std::cos(theta), sth = std::sin(theta);
  if (variant == 0) {
    *mode = 0;
    *h = w / 2.0;
    *cr = r * cth;
    *ci = r * sth;
  } else {
    *mode = 1;
    double s = (w / 4.0) * r;
    *h = 0.0;
    *cr = s * cth;
    *ci = s * (variant == 1 ? sth : -sth);
  }
}

int fb_accumulate(fb_ctx* c, int variant, int n, int m, const double* xr, const double* xi, int64_t ldx,
                  double* qr, double* qi, int64_t ldq, double w, double r, double theta) {
  CTX_GUARD(c);
  if (variant < 0 || variant > 2) return FB_ERR_ARG;
  int mode;
  double h, cr, ci;
  acc_coeffs(variant, w, r, theta, &mode, &h, &cr, &ci);
  return set_err(c, fb::accumulate_launch(mode, n, m, xr, xi, ldx, qr, qi, ldq, h, cr, ci, c->stream),
                 "accumulate");
}

int fb_accumulate_terms(fb_ctx* c, int count, const int* variant, const double* w, double r, const double* theta,
                        const double* const* xr, const double* const* xi, int n, int m, int64_t ldx, double* qr,
                        double* qi, int64_t ldq) {
  CTX_GUARD(c);
  if (count < 0 || count > fb::kMaxAccTerms) return FB_ERR_ARG;
  fb::AccTerms t{};
  t.count = count;
  for (int k = 0; k < count; ++k) {
    if (variant[k] < 0 || variant[k] > 2 || (variant[k] == 0) != (variant[0] == 0)) return FB_ERR_ARG;
    acc_coeffs(variant[k], w[k], r, theta[k], &t.mode[k], &t.h[k], &t.cr[k], &t.ci[k]);
    t.xr[k] = xr[k];
    t.xi[k] = xi[k];
  }
  return set_err(c, fb::accumulate_terms_launch(t, n, m, ldx, qr, qi, ldq, c->stream), "accumulate_terms");
}

int fb_gemm(fb_ctx* c, int cplx, char opa, char opb, int m, int n, int k, double ar, double ai,
            const double* are, const double* aim, int64_t lda, const double* bre, const double* bim,
            int64_t ldb, double br, double bi, double* cre, double* cim, int64_t ldc) {
  CTX_GUARD(c);
  if (m < 0 || n < 0 || k < 0 || !cre || (cplx && !cim)) return FB_ERR_ARG;
  fb::GemmParams p;
  p.m = m; p.n = n; p.k = k;
  p.a = make_op(opa, are, cplx ? aim : nullptr, lda);
  p.b = make_op(opb, bre, cplx ? bim : nullptr, ldb);
  p.cre = cre; p.cim = cplx ? cim : nullptr; p.cs0 = ldc; p.cs1 = 1;
  p.alpha_re = ar; p.alpha_im = cplx ? ai : 0.0; p.beta_re = br; p.beta_im = cplx ? bi : 0.0;
  p.splits = fb::gemm_pick_splits(m, n, k);
  p.ws = nullptr;
  p.kchunk = 0;
  if (p.splits > 1) {
    int r = ensure_scratch(c, fb::gemm_workspace_bytes(cplx, m, n, p.splits));
    if (r) return r;
    p.ws = (double*)c->scratch;
  }
  return set_err(c, fb::gemm_launch(cplx, p, c->stream), "gemm");
}

int fb_symmetrize(fb_ctx* c, int m, double* re, double* im, int64_t ld) {
  CTX_GUARD(c);
  return set_err(c, fb::symmetrize_launch(m, re, im, ld, c->stream), "symmetrize");
}

int fb_residuals(fb_ctx* c, int n, int m, const double* axr, const double* axi, const double* bxr,
                 const double* bxi, int64_t ld, const double* lam, double scale, double* res) {
  CTX_GUARD(c);
  int r = ensure_scratch(c, fb::residual_scratch_bytes(n, m));
  if (r) return r;
  return set_err(c, fb::residual_launch(n, m, axr, axi, bxr, bxi, ld, lam, scale, res,
                                        (double*)c->scratch, c->stream),
                 "residuals");
}

int fb_residual_sums(fb_ctx* c, int n, int m, const double* axr, const double* axi, const double* bxr,
                     const double* bxi, int64_t ld, const double* lam, double scale, double* sums) {
  CTX_GUARD(c);
  if (n < 0 || m < 0 || !sums) return FB_ERR_ARG;
  int r = ensure_scratch(c, fb::residual_scratch_bytes(n > 0 ? n : 1, m));
  if (r) return r;
  return set_err(c, fb::residual_sums_launch(n, m, axr, axi, bxr, bxi, ld, lam, scale, sums,
                                             (double*)c->scratch, c->stream),
                 "residual_sums");
}

int fb_chol_check(fb_ctx* c, int m, const double* bre, const double* bim, int64_t ld, int* fail) {
  CTX_GUARD(c);
  if (m <= 0 || !fail) return FB_ERR_ARG;
  const bool cl = fb::reduced_cluster_ok(m, bim != nullptr);
  int r = ensure_scratch(c, cl ? fb::reduced_cluster_scratch_bytes(m) : fb::reduced_scratch_bytes(m));
  if (r) return r;
  cudaError_t e = cl ? fb::reduced_cluster_launch(m, bre, bim, bre, bim, ld, nullptr, nullptr, nullptr, 0,
                                                  c->dev_word, (double*)c->scratch, 1, c->stream)
                     : fb::chol_check_launch(m, bre, bim, ld, c->dev_word, (double*)c->scratch, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->host_word, c->dev_word, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_err(c, e, "chol_check");
  *fail = c->host_word[0];
  return FB_OK;
}

int fb_reduced_eig(fb_ctx* c, int m, const double* are, const double* aim, const double* bre,
                   const double* bim, int64_t ld, double* eps, double* phre, double* phim, int64_t ldphi,
                   int* status) {
  CTX_GUARD(c);
  if (m <= 0 || !status || !eps || !phre) return FB_ERR_ARG;
  const bool cl = fb::reduced_cluster_ok(m, bim != nullptr) && !getenv("FB_REDUCED_QL");
  int r = ensure_scratch(c, cl ? fb::reduced_cluster_scratch_bytes(m) : fb::reduced_scratch_bytes(m));
  if (r) return r;
  cudaError_t e = cl ? fb::reduced_cluster_launch(m, are, aim, bre, bim, ld, eps, phre, phim, ldphi,
                                                  c->dev_word, (double*)c->scratch, 0, c->stream)
                     : fb::reduced_eig_launch(m, are, aim, bre, bim, ld, eps, phre, phim, ldphi, c->dev_word,
                                              (double*)c->scratch, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->host_word, c->dev_word, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return set_err(c, e, "reduced_eig");
  *status = c->host_word[0];
  return *status == 0 ? FB_OK : fb::FB_ERR_REDUCED;
}

int fb_pack(fb_ctx* c, int n, int m, const double* z, int64_t ldz, double* re, double* im, int64_t ld,
            int to_planar) {
  CTX_GUARD(c);
  return set_err(c, fb::pack_launch(n, m, z, ldz, re, im, ld, to_planar, c->stream), "pack");
}

int fb_band_matvec(fb_ctx* c, int n, int kl, int m, const double* fbr, const double* fbi, int64_t ldb,
                   const double* xr, const double* xi, int64_t ldx, double* yr, double* yi, int64_t ldy) {
  CTX_GUARD(c);
  if (n < 0 || kl < 0 || m < 0 || !fbr || !xr || !yr) return FB_ERR_ARG;
  return set_err(c, fb::band_matvec_launch(n, kl, m, fbr, fbi, ldb, xr, xi, ldx, yr, yi, ldy, c->stream),
                 "band_matvec");
}

int fb_band_factor(fb_ctx* c, int n, int kl, double zr, double zi, const double* far_, const double* fai,
                   const double* fbr, const double* fbi, int64_t ldb, double* fr, double* fi, int* ipiv,
                   int* info) {
  CTX_GUARD(c);
  if (n < 0 || kl < 0 || !far_ || !fr || !fi || !ipiv || !info) return FB_ERR_ARG;
  const int big = INT_MAX;
  cudaError_t e = cudaMemcpyAsync(info, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream);
  if (e != cudaSuccess) return set_err(c, e, "band info init");
  return set_err(c, fb::band_factor_launch(n, kl, zr, zi, far_, fai, fbr, fbi, ldb, fr, fi, ipiv, info,
                                           c->stream),
                 "band_factor");
}

int fb_band_solve(fb_ctx* c, int n, int kl, int nrhs, const double* fr, const double* fi, const int* ipiv,
                  int adjoint, double* xr, double* xi, int64_t ldx) {
  CTX_GUARD(c);
  if (n < 0 || kl < 0 || nrhs < 0 || !fr || !xr || !xi) return FB_ERR_ARG;
  return set_err(c, fb::band_solve_launch(n, kl, nrhs, fr, fi, ipiv, adjoint, xr, xi, ldx, c->stream),
                 "band_solve");
}

int64_t fb_band_aux_doubles(int n, int kl) {
  if (n <= 0 || !fb::band_spike_ok(kl)) return 0;
  return (int64_t)fb::band_spike_aux_doubles(n, kl);
}

int fb_band_factor_batched(fb_ctx* c, int count, int n, int kl, const double* zr, const double* zi,
                           const double* far_, const double* fai, const double* fbr, const double* fbi,
                           int64_t ldb, double* fr, double* fi, int64_t fs, int* ipiv, int64_t ps, double* aux,
                           int64_t as, int* info) {
  CTX_GUARD(c);
  if (count < 0 || count > 64 || n < 0 || !fb::band_spike_ok(kl) || !zr || !zi || !far_ || !fr || !fi ||
      !ipiv || !aux || !info)
    return FB_ERR_ARG;
  return set_err(c, fb::band_spike_factor(count, n, kl, zr, zi, far_, fai, fbr, fbi, ldb, fr, fi, fs, ipiv, ps,
                                          aux, as, info, c->stream),
                 "band_factor_batched");
}

int fb_band_solve_batched(fb_ctx* c, int count, int n, int kl, int nrhs, const double* fr, const double* fi,
                          int64_t fs, const int* ipiv, int64_t ps, const double* aux, int64_t as, double* xr,
                          double* xi, int64_t ldx, int64_t xs) {
  CTX_GUARD(c);
  if (count < 0 || count > 64 || n < 0 || nrhs < 0 || !fb::band_spike_ok(kl) || !fr || !fi || !ipiv || !aux ||
      !xr || !xi)
    return FB_ERR_ARG;
  int r = ensure_scratch(c, sizeof(double) * fb::band_spike_solve_scratch_doubles(n, kl, nrhs, count));
  if (r) return r;
  return set_err(c, fb::band_spike_solve(count, n, kl, nrhs, fr, fi, fs, ipiv, ps, aux, as, xr, xi, ldx, xs,
                                         (double*)c->scratch, c->stream),
                 "band_solve_batched");
}

int fb_band_solve_batched_rhs(fb_ctx* c, int count, int n, int kl, int nrhs, const double* fr, const double* fi,
                              int64_t fs, const int* ipiv, int64_t ps, const double* aux, int64_t as,
                              const double* yr, const double* yi, int64_t ldy, int64_t ys, double* xr, double* xi,
                              int64_t ldx, int64_t xs) {
  CTX_GUARD(c);
  if (count < 0 || count > 64 || n < 0 || nrhs < 0 || !fb::band_spike_ok(kl) || !fr || !fi || !ipiv || !aux ||
      !xr || !xi || !yr)
    return FB_ERR_ARG;
  int r = ensure_scratch(c, sizeof(double) * fb::band_spike_solve_scratch_doubles(n, kl, nrhs, count));
  if (r) return r;
  return set_err(c, fb::band_spike_solve(count, n, kl, nrhs, fr, fi, fs, ipiv, ps, aux, as, xr, xi, ldx, xs,
                                         (double*)c->scratch, c->stream, yr, yi, ldy, ys),
                 "band_solve_batched_rhs");
}

int fb_band_solve_accumulate(fb_ctx* c, int count, int n, int kl, int nrhs, const double* fr, const double* fi,
                             int64_t fs, const int* ipiv, int64_t ps, const double* aux, int64_t as,
                             const double* yr, const double* yi, int64_t ldy, double* xr, double* xi, int64_t ldx,
                             int64_t xs, int nterms, const int* item, const int* variant, const double* w, double r,
                             const double* theta, double* qr, double* qi, int64_t ldq) {
  CTX_GUARD(c);
  if (count < 0 || count > 64 || n < 0 || nrhs < 0 || !fb::band_spike_ok(kl) || !fr || !fi || !ipiv || !aux ||
      !xr || !xi || !yr || !qr || nterms < 0 || nterms > fb::kMaxAccTerms || !item || !variant || !w || !theta)
    return FB_ERR_ARG;
  fb::AccTerms t{};
  t.count = nterms;
  for (int k = 0; k < nterms; ++k) {
    if (variant[k] < 0 || variant[k] > 2 || (variant[k] == 0) != (variant[0] == 0)) return FB_ERR_ARG;
    if (variant[k] != 0 && !qi) return FB_ERR_ARG;
    acc_coeffs(variant[k], w[k], r, theta[k], &t.mode[k], &t.h[k], &t.cr[k], &t.ci[k]);
  }
  int rc = ensure_scratch(c, sizeof(double) * fb::band_spike_solve_scratch_doubles(n, kl, nrhs, count));
  if (rc) return rc;
  return set_err(c, fb::band_spike_solve_accumulate(count, n, kl, nrhs, fr, fi, fs, ipiv, ps, aux, as, xr, xi, ldx,
                                                    xs, (double*)c->scratch, c->stream, yr, yi, ldy, t, item, qr,
                                                    qi, ldq),
                 "band_solve_accumulate");
}

// Debug only (not part of the ABI header): partition size target of the
// SPIKE band path (tests force many partitions at small n); returns P.
int fb_debug_band_part_target(int target, int n, int kl) {
  fb::band_spike_set_part_target(target);
  return fb::band_spike_parts(n, kl);
}

// Debug only (not part of the ABI header): cycles per panel phase, CTA 0 / thread 0.
int fb_debug_panel_profile(unsigned long long* out8) {
  fb::panel_profile_read(out8);
  return FB_OK;
}

// Debug only: CTA 0 of the cluster panels, summed over launches: wall ns
// (globaltimer), SM cycles (clock64), launch count.
int fb_debug_panel_wall(unsigned long long* out4) {
  fb::panel_wall_read(out4);
  return FB_OK;
}

// Debug only (FB_PANEL_EVENTS=1): summed event time around the panel launches.
double fb_debug_panel_events(int* count) { return fb::panel_events_read_ms(count); }

int fb_debug_reduced_profile(unsigned long long* out8) {
  // single-CTA counters, or the cluster kernel's when it ran
  unsigned long long c8[8];
  fb::reduced_profile_read(out8);
  fb::reduced_cluster_profile_read(c8);
  bool any = false;
  for (int k = 0; k < 8; ++k) any |= c8[k] != 0;
  if (any)
    for (int k = 0; k < 8; ++k) out8[k] = c8[k];
  return FB_OK;
}


// ---- CSR backend -------------------------------------------------------------------------------

int fb_csr_matvec(fb_ctx* c, int n, int m, const int64_t* indptr, const int64_t* indices, const double* vr,
                  const double* vi, const double* xr, const double* xi, int64_t ldx, double* yr, double* yi,
                  int64_t ldy, const int64_t* row_order) {
  CTX_GUARD(c);
  if (n < 0 || m < 0 || !indptr || !xr || !yr) return FB_ERR_ARG;
  if ((vi || xi) && !yi) return FB_ERR_ARG;
  return set_err(c,
                 fb::csr_spmm_launch(n, m, reinterpret_cast<const long long*>(indptr),
                                     reinterpret_cast<const long long*>(indices), vr, vi, xr, xi, ldx, yr, yi, ldy,
                                     reinterpret_cast<const long long*>(row_order), c->stream),
                 "csr_matvec");
}

int fb_permute_rows(fb_ctx* c, int n, int m, const int64_t* perm, const double* sr, const double* si, int64_t lds,
                    double* dr, double* di, int64_t ldd) {
  CTX_GUARD(c);
  if (n < 0 || m < 0 || !perm || !sr || !dr || (!si) != (!di)) return FB_ERR_ARG;
  return set_err(c,
                 fb::gather_rows_launch(n, m, reinterpret_cast<const long long*>(perm), sr, si, lds, dr, di, ldd,
                                         c->stream),
                 "permute_rows");
}

int64_t fb_bicgstab_workspace_doubles(int n, int m, int64_t ld) {
  if (n < 0 || m < 0 || ld < m) return -1;
  return (int64_t)fb::bicgstab_workspace_doubles(n, m, ld);
}

int fb_bicgstab(fb_ctx* c, int phase, int n, int m, const int64_t* indptr, const int64_t* indices, const double* sr,
                const double* si, const double* dr, const double* di, const double* br, const double* bi,
                int64_t ldb, double* xr, double* xi, int64_t ldx, double tol, int maxiter, int iters, double* work,
                int64_t ld, int* istate, const int64_t* row_order) {
  CTX_GUARD(c);
  if (n <= 0 || m <= 0 || !indptr || !indices || !sr || !si || !dr || !di || !br || !xr || !xi || !work ||
      !istate || ldx != ld || ld < m || (phase != 0 && phase != 1) || iters < 0)
    return FB_ERR_ARG;
  return set_err(c,
                 fb::bicgstab_launch(phase, n, m, reinterpret_cast<const long long*>(indptr),
                                     reinterpret_cast<const long long*>(indices), sr, si, dr, di, br, bi, ldb, xr,
                                     xi, ldx, tol, maxiter, iters, work, ld, istate,
                                     reinterpret_cast<const long long*>(row_order), c->stream),
                 "bicgstab");
}

}  // extern "C"
