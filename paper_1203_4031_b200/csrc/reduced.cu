// Reduced (M0 x M0) generalized Hermitian eigensolver, on the GPU.
//
// Restates reduced.py:22-218 step for step so the Ritz values follow the
// reference algorithm:
//   spd_factor (Cholesky with 1-based failing-pivot index)       reduced.py:22-40
//   C = L^-1 A L^-H, then C <- (C + C^H)/2                        reduced.py:209-212
//   Householder tridiagonalisation with accumulated V             reduced.py:65-114
//   complex phase folding of the subdiagonal into V               reduced.py:102-113
//   implicit QL with Wilkinson shifts, <= 30 sweeps / eigenvalue  reduced.py:117-172
//   stable ascending sort, Phi = L^-H Y                           reduced.py:180-185, 213-218
//
// One CTA of 1024 threads does the whole solve (M0 <= 512 here).  Every
// O(M0^3) stage is written right-looking — each of the M0 sequential steps is
// an elementwise update spread over all threads with coalesced row-major
// accesses — so a step costs a couple of barriers and one L2 round trip
// instead of a dependent chain of loads.  The O(M0^2) QL recurrences run on
// one thread; their rotation sequence is applied by all threads to
// contiguous rows of V^T.  Working arrays live in a global scratch
// (L2-resident for M0 <= 512).
#include <cstdlib>

#include "common.cuh"
#include "misc.cuh"

namespace fb {

namespace {

constexpr int RT = 1024;  // threads
constexpr int NWARP = RT / 32;
// rows over warps, columns over lanes: no integer division, coalesced rows
#define FOR2D(i, rows, j, cols)                              \
  for (int i = threadIdx.x >> 5; i < (rows); i += NWARP)     \
    for (int j = threadIdx.x & 31; j < (cols); j += 32)

__device__ double block_sum(double x, double* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

struct RArgs {
  int m;
  const double *are, *aim, *bre, *bim;
  long long ld;
  double* eps;
  double *phre, *phim;
  long long ldphi;
  int* status;
  double* ws;
  int check_only;
  int method;  // 0: bisection + inverse iteration, 1: implicit QL (reduced.py:117-172)
};

// Sturm count: #eigenvalues of T(d, e) below x (LDL^T negative pivots).
__device__ int sturm_count(int m, const double* d, const double* e2, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) <= pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < m; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) <= pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// Eigenpairs of the symmetric tridiagonal T (diag d[m], off-diagonal e[m-1]).
// eps[k] = k-th smallest eigenvalue, Zt[k*m + i] = i-th entry of its unit
// eigenvector.  Work: Wk (6m doubles per eigenvalue) and the block scratch sh.
__device__ void tridiag_bisect_invit(int m, const double* d, const double* e, double* eps, double* Zt,
                                     double* Wk, double* sh) {
  const int tid = threadIdx.x;
  const double ulp = 2.220446049250313e-16;
  // Gershgorin bounds, ||T||_1 and the pivot floor (LAPACK dstebz)
  __shared__ double s_gl, s_gu, s_tn, s_pm;
  if (tid == 0) {
    double gl = d[0], gu = d[0], tn = 0.0, emax2 = 0.0;
    for (int i = 0; i < m; ++i) {
      const double el = i > 0 ? fabs(e[i - 1]) : 0.0, er = i + 1 < m ? fabs(e[i]) : 0.0;
      gl = fmin(gl, d[i] - el - er);
      gu = fmax(gu, d[i] + el + er);
      tn = fmax(tn, fabs(d[i]) + el + er);
      if (i + 1 < m) emax2 = fmax(emax2, e[i] * e[i]);
    }
    const double pad = 2.0 * ulp * fmax(fabs(gl), fabs(gu)) + 1e-300;
    s_gl = gl - pad;
    s_gu = gu + pad;
    s_tn = tn > 0.0 ? tn : 1.0;
    s_pm = fmax(1e-290, ulp * ulp * emax2);
  }
  // e^2 into the block scratch area past the reduction slots
  double* e2 = Wk + (size_t)m * 6 * m;   // [m]
  for (int i = tid; i + 1 < m; i += blockDim.x) e2[i] = e[i] * e[i];
  __syncthreads();
  const double gl = s_gl, gu = s_gu, tnorm = s_tn, pivmin = s_pm;
  for (int k = tid; k < m; k += blockDim.x) {
    double lo = gl, hi = gu;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      if (hi - lo <= 2.0 * ulp * fmax(fabs(lo), fabs(hi)) + pivmin) break;
      if (sturm_count(m, d, e2, mid, pivmin) > k) hi = mid; else lo = mid;
    }
    eps[k] = 0.5 * (lo + hi);
  }
  __syncthreads();
  // inverse iteration; a cluster (gap <= 1e-3 ||T||) is handled by its first thread
  const double ortol = 1e-3 * tnorm;
  const double tiny = ulp * tnorm;
  for (int k = tid; k < m; k += blockDim.x) {
    if (k > 0 && eps[k] - eps[k - 1] <= ortol) continue;   // not a cluster leader
    int kend = k + 1;
    while (kend < m && eps[kend] - eps[kend - 1] <= ortol) ++kend;
    double* W = Wk + (size_t)k * 6 * m;
    double *u0 = W, *u1 = W + m, *u2 = W + 2 * m, *lm = W + 3 * m, *sw = W + 4 * m, *y = W + 5 * m;
    double lam = 0.0;
    for (int j = k; j < kend; ++j) {
      // separate (nearly) coincident eigenvalues by 10 ulp of the eigenvalue
      // itself, as LAPACK dstein does: a norm-relative step would move the
      // small Ritz values of a graded (ill-conditioned B_Q) pencil far off
      const double pert = 10.0 * ulp * fabs(eps[j]);
      lam = (j > k && eps[j] - lam < pert) ? lam + pert : eps[j];
      // LU with partial pivoting of T - lam I (U has two superdiagonals)
      double c0 = d[0] - lam, c1 = m > 1 ? e[0] : 0.0, c2 = 0.0;
      for (int i = 0; i + 1 < m; ++i) {
        const double n0 = e[i], n1 = d[i + 1] - lam, n2 = i + 2 < m ? e[i + 1] : 0.0;
        if (fabs(c0) >= fabs(n0)) {
          if (c0 == 0.0) c0 = tiny;
          const double l = n0 / c0;
          u0[i] = c0; u1[i] = c1; u2[i] = c2; lm[i] = l; sw[i] = 0.0;
          c0 = n1 - l * c1;
          c1 = n2 - l * c2;
          c2 = 0.0;
        } else {
          const double l = c0 / n0;
          u0[i] = n0; u1[i] = n1; u2[i] = n2; lm[i] = l; sw[i] = 1.0;
          const double t0 = c1 - l * n1, t1 = c2 - l * n2;
          c0 = t0;
          c1 = t1;
          c2 = 0.0;
        }
      }
      if (fabs(c0) < tiny) c0 = c0 < 0.0 ? -tiny : tiny;
      u0[m - 1] = c0; u1[m - 1] = 0.0; u2[m - 1] = 0.0;
      for (int i = 0; i + 1 < m; ++i)
        if (fabs(u0[i]) < tiny) u0[i] = u0[i] < 0.0 ? -tiny : tiny;
      // deterministic start vector
      for (int i = 0; i < m; ++i) {
        unsigned long long z = 0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1) + (unsigned long long)j * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 31)) * 0x94D049BB133111EBull;
        y[i] = ((double)(z >> 11) * 0x1p-53) - 0.5;
      }
      double* x = Zt + (size_t)j * m;
      for (int iter = 0; iter < 3; ++iter) {
        for (int i = 0; i + 1 < m; ++i) {   // apply L (with interchanges)
          if (sw[i] != 0.0) {
            const double t = y[i];
            y[i] = y[i + 1];
            y[i + 1] = t;
          }
          y[i + 1] -= lm[i] * y[i];
        }
        for (int i = m - 1; i >= 0; --i) {  // U back substitution
          double v = y[i];
          if (i + 1 < m) v -= u1[i] * y[i + 1];
          if (i + 2 < m) v -= u2[i] * y[i + 2];
          y[i] = v / u0[i];
        }
        for (int q = k; q < j; ++q) {       // re-orthogonalise inside the cluster
          const double* zq = Zt + (size_t)q * m;
          double dot = 0.0;
          for (int i = 0; i < m; ++i) dot += zq[i] * y[i];
          for (int i = 0; i < m; ++i) y[i] -= dot * zq[i];
        }
        double mx = 0.0;
        for (int i = 0; i < m; ++i) mx = fmax(mx, fabs(y[i]));
        if (mx == 0.0) mx = 1.0;
        double nrm = 0.0;
        for (int i = 0; i < m; ++i) {
          y[i] /= mx;
          nrm += y[i] * y[i];
        }
        nrm = sqrt(nrm);
        for (int i = 0; i < m; ++i) y[i] /= nrm;
      }
      for (int i = 0; i < m; ++i) x[i] = y[i];
    }
  }
}

__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double& cr, double& ci) {
  cr = ar * br - ai * bi;
  ci = ar * bi + ai * br;
}

__device__ unsigned long long g_reduced_prof[8];
#define RPROBE(k)                                                                   \
  do {                                                                              \
    if (threadIdx.x == 0) {                                                         \
      long long _n = clock64();                                                     \
      atomicAdd(&g_reduced_prof[k], (unsigned long long)(_n - _rt));                \
      _rt = _n;                                                                     \
    }                                                                               \
  } while (0)

template <bool CPLX>
__global__ void __launch_bounds__(RT, 1) reduced_kernel(RArgs a) {
  long long _rt = clock64();
  const int m = a.m, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t mm = (size_t)m * m;
  double* Lr = a.ws;      // Cholesky factor (lower), in place of a copy of B
  double* Li = Lr + mm;
  double* Cr = Li + mm;   // working matrix (row-major)
  double* Ci = Cr + mm;
  double* Tr = Ci + mm;   // scratch / V (row-major during Householder)
  double* Ti = Tr + mm;
  double* Vr = Ti + mm;   // V^T for the QL rotations: Vr[c*m + r] = V[r][c]
  double* Vi = Vr + mm;
  double* ur = Vi + mm;
  double* ui = ur + m;
  double* pr = ui + m;
  double* pi = pr + m;
  double* wr = pi + m;
  double* wi = wr + m;
  double* Zt = wi + m;            // eigenvectors of T, one row per eigenvalue
  double* Wk = Zt + mm;           // inverse-iteration work, 6m doubles per eigenvalue
  extern __shared__ double shd[];
  double* d = shd;           // [m]
  double* ee = d + m;        // [m]
  double* rc = ee + m;       // rotation cosines [m]
  double* rs = rc + m;       // rotation sines [m]
  double* sh = rs + m;       // reduction scratch [40]
  __shared__ int s_int[4];
  __shared__ double s_val[2];


  // 1. Cholesky L L^H = B, right-looking on a copy (reduced.py:22-40); the
  //    lower triangle of (Lr, Li) ends up holding L, the rest is zeroed.
  FOR2D(i, m, j, m) {
    Lr[(size_t)i * m + j] = a.bre[i * a.ld + j];
    if (CPLX) Li[(size_t)i * m + j] = a.bim[i * a.ld + j];
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (tid == 0) {
      const double dj = Lr[(size_t)j * m + j];
      s_int[0] = (!(dj > 0.0) || !isfinite(dj)) ? j + 1 : 0;
      s_val[0] = sqrt(dj);
    }
    __syncthreads();
    if (s_int[0]) {
      if (tid == 0) *a.status = s_int[0];
      return;
    }
    const double ljj = s_val[0];
    for (int i = j + 1 + tid; i < m; i += RT) {
      Lr[(size_t)i * m + j] /= ljj;
      if (CPLX) Li[(size_t)i * m + j] /= ljj;
    }
    if (tid == 0) {
      Lr[(size_t)j * m + j] = ljj;
      if (CPLX) Li[(size_t)j * m + j] = 0.0;
    }
    __syncthreads();
    // trailing update W[i][k] -= L[i][j] conj(L[k][j]), j < k <= i
    const int t = m - j - 1;
    FOR2D(ii, t, kk, ii + 1) {
      const int i = j + 1 + ii, k = j + 1 + kk;
      const double xr = Lr[(size_t)i * m + j], yr = Lr[(size_t)k * m + j];
      if (CPLX) {
        const double xi = Li[(size_t)i * m + j], yi = -Li[(size_t)k * m + j];
        Lr[(size_t)i * m + k] -= xr * yr - xi * yi;
        Li[(size_t)i * m + k] -= xr * yi + xi * yr;
      } else {
        Lr[(size_t)i * m + k] -= xr * yr;
      }
    }
    __syncthreads();
  }
  FOR2D(i, m, j, m) {  // strictly upper part of L is zero
    if (j > i) {
      Lr[(size_t)i * m + j] = 0.0;
      if (CPLX) Li[(size_t)i * m + j] = 0.0;
    }
  }
  __syncthreads();
  RPROBE(0);
  if (!a.check_only) {
    // finiteness after the Cholesky: a pivot failure wins (the caller shrinks
    // M0, kernel.py:385-400), otherwise non-finite input is the reduced solver
    // error (reduced.py:203-204)
    int bad = 0;
    FOR2D(i, m, j, m) {
      double x = a.are[i * a.ld + j] + a.bre[i * a.ld + j];
      if (CPLX) x += a.aim[i * a.ld + j] + a.bim[i * a.ld + j];
      if (!isfinite(x)) bad = 1;
    }
    if (__syncthreads_or(bad)) {
      if (tid == 0) *a.status = -2;
      return;
    }
    if (m == 1) {  // reduced.py:205-210
      if (tid == 0) {
        const double b00 = a.bre[0];
        a.eps[0] = a.are[0] / b00;
        a.phre[0] = 1.0 / sqrt(b00);
        if (CPLX) a.phim[0] = 0.0;
        *a.status = 0;
      }
      return;
    }
  }
  if (a.check_only) {
    if (tid == 0) *a.status = 0;
    return;
  }

  // right-looking forward substitution X <- L^-1 X in place (X row-major m x m)
  auto lower_solve = [&](double* Xr, double* Xi) {
    for (int i = 0; i < m; ++i) {
      const double dr = Lr[(size_t)i * m + i];
      for (int c = tid; c < m; c += RT) {
        Xr[(size_t)i * m + c] /= dr;
        if (CPLX) Xi[(size_t)i * m + c] /= dr;
      }
      __syncthreads();
      const int t = m - i - 1;
      FOR2D(rr, t, c, m) {
        const int r = i + 1 + rr;
        const double lr = Lr[(size_t)r * m + i], xr = Xr[(size_t)i * m + c];
        if (CPLX) {
          const double li = Li[(size_t)r * m + i], xi = Xi[(size_t)i * m + c];
          Xr[(size_t)r * m + c] -= lr * xr - li * xi;
          Xi[(size_t)r * m + c] -= lr * xi + li * xr;
        } else {
          Xr[(size_t)r * m + c] -= lr * xr;
        }
      }
      __syncthreads();
    }
  };

  // 2. C = L^-1 A L^-H  (reduced.py:209-212)
  FOR2D(i, m, j, m) {
    Cr[(size_t)i * m + j] = a.are[i * a.ld + j];
    if (CPLX) Ci[(size_t)i * m + j] = a.aim[i * a.ld + j];
  }
  __syncthreads();
  lower_solve(Cr, Ci);                       // W = L^-1 A
  FOR2D(j, m, i, m) {                        // T = W^H (coalesced writes)
    Tr[(size_t)j * m + i] = Cr[(size_t)i * m + j];
    if (CPLX) Ti[(size_t)j * m + i] = -Ci[(size_t)i * m + j];
  }
  __syncthreads();
  lower_solve(Tr, Ti);                       // X = L^-1 W^H
  FOR2D(i, m, j, m) {                        // C = X^H, then (C + C^H)/2
    const double xr = Tr[(size_t)j * m + i], yr = Tr[(size_t)i * m + j];
    Cr[(size_t)i * m + j] = 0.5 * (xr + yr);
    if (CPLX) Ci[(size_t)i * m + j] = 0.5 * (-Ti[(size_t)j * m + i] + Ti[(size_t)i * m + j]);
  }
  __syncthreads();
  // V = I, row-major in T during the Householder phase
  FOR2D(i, m, j, m) {
    Tr[(size_t)i * m + j] = (i == j) ? 1.0 : 0.0;
    if (CPLX) Ti[(size_t)i * m + j] = 0.0;
  }
  __syncthreads();

  RPROBE(1);
  // 3. Householder tridiagonalisation (reduced.py:73-100)
  for (int k = 0; k + 2 < m; ++k) {
    const int len = m - k - 1;
    double part = 0.0;
    for (int i = tid; i < len; i += RT) {
      double xr = Cr[(size_t)(k + 1 + i) * m + k], xi = CPLX ? Ci[(size_t)(k + 1 + i) * m + k] : 0.0;
      ur[i] = xr;
      if (CPLX) ui[i] = xi;
      part += xr * xr + xi * xi;
    }
    double xnorm = sqrt(block_sum(part, sh));
    if (xnorm == 0.0) continue;
    double x0r = Cr[(size_t)(k + 1) * m + k], x0i = CPLX ? Ci[(size_t)(k + 1) * m + k] : 0.0;
    double ax0 = CPLX ? hypot(x0r, x0i) : fabs(x0r);
    double phr = 1.0, phi_ = 0.0;
    if (ax0 != 0.0) {
      phr = x0r / ax0;
      phi_ = x0i / ax0;
    }
    const double alr = -phr * xnorm, ali = -phi_ * xnorm;
    if (tid == 0) {
      ur[0] = x0r - alr;
      if (CPLX) ui[0] = x0i - ali;
    }
    __syncthreads();
    part = 0.0;
    for (int i = tid; i < len; i += RT) {
      double xr = ur[i], xi = CPLX ? ui[i] : 0.0;
      part += xr * xr + xi * xi;
    }
    double unorm = sqrt(block_sum(part, sh));
    if (unorm == 0.0) continue;
    for (int i = tid; i < len; i += RT) {
      ur[i] /= unorm;
      if (CPLX) ui[i] /= unorm;
    }
    __syncthreads();
    // p = 2 * sub @ u and w = V[:, k+1:] @ u (one warp per row, lanes along the row)
    for (int i = warp; i < len + m; i += RT / 32) {
      const bool isp = i < len;
      const double* rowr = isp ? Cr + (size_t)(k + 1 + i) * m + k + 1 : Tr + (size_t)(i - len) * m + k + 1;
      const double* rowi = isp ? Ci + (size_t)(k + 1 + i) * m + k + 1 : Ti + (size_t)(i - len) * m + k + 1;
      double sr = 0.0, si = 0.0;
      for (int j = lane; j < len; j += 32) {
        if (CPLX) {
          sr += rowr[j] * ur[j] - rowi[j] * ui[j];
          si += rowr[j] * ui[j] + rowi[j] * ur[j];
        } else {
          sr += rowr[j] * ur[j];
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        si += __shfl_xor_sync(0xffffffffu, si, o);
      }
      if (lane == 0) {
        if (isp) {
          pr[i] = 2.0 * sr;
          if (CPLX) pi[i] = 2.0 * si;
        } else {
          wr[i - len] = sr;
          if (CPLX) wi[i - len] = si;
        }
      }
    }
    __syncthreads();
    part = 0.0;  // kappa = Re(u^H p)
    for (int i = tid; i < len; i += RT) part += ur[i] * pr[i] + (CPLX ? ui[i] * pi[i] : 0.0);
    const double kap2 = 2.0 * block_sum(part, sh);
    // sub -= p u^H ; sub -= u p^H ; sub += 2 kappa u u^H ; V[:, k+1:] -= 2 w u^H
    for (int i = warp; i < len + m; i += NWARP) {
      const bool isc = i < len;
      for (int j = lane; j < len; j += 32) {
        if (isc) {
          const size_t o = (size_t)(k + 1 + i) * m + k + 1 + j;
          if (CPLX) {
            double tr, ti;
            double sr = Cr[o], si = Ci[o];
            cmul(pr[i], pi[i], ur[j], -ui[j], tr, ti);
            sr -= tr;
            si -= ti;
            cmul(ur[i], ui[i], pr[j], -pi[j], tr, ti);
            sr -= tr;
            si -= ti;
            cmul(ur[i], ui[i], ur[j], -ui[j], tr, ti);
            sr += kap2 * tr;
            si += kap2 * ti;
            Cr[o] = sr;
            Ci[o] = si;
          } else {
            double s_ = Cr[o];
            s_ -= pr[i] * ur[j];
            s_ -= ur[i] * pr[j];
            s_ += kap2 * (ur[i] * ur[j]);
            Cr[o] = s_;
          }
        } else {
          const int r = i - len;
          const size_t o = (size_t)r * m + k + 1 + j;
          if (CPLX) {
            double tr, ti;
            cmul(wr[r], wi[r], ur[j], -ui[j], tr, ti);
            Tr[o] -= 2.0 * tr;
            Ti[o] -= 2.0 * ti;
          } else {
            Tr[o] -= 2.0 * (wr[r] * ur[j]);
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      Cr[(size_t)(k + 1) * m + k] = alr;
      if (CPLX) Ci[(size_t)(k + 1) * m + k] = ali;
    }
    __syncthreads();
  }

  RPROBE(2);
  // 4. d, e and (complex) phase folding (reduced.py:101-113)
  for (int i = tid; i < m; i += RT) d[i] = Cr[(size_t)i * m + i];
  __syncthreads();
  if (tid == 0) {
    double fr = 1.0, fi = 0.0;  // running phase phi[j]
    wr[0] = 1.0;
    if (CPLX) wi[0] = 0.0;
    for (int j = 0; j + 1 < m; ++j) {
      double sr = Cr[(size_t)(j + 1) * m + j];
      if (CPLX) {
        double si = Ci[(size_t)(j + 1) * m + j];
        double mag = hypot(sr, si);
        if (mag != 0.0) {
          double nr, ni;
          cmul(fr, fi, sr / mag, si / mag, nr, ni);
          fr = nr;
          fi = ni;
        }
        ee[j] = mag;
        wr[j + 1] = fr;
        wi[j + 1] = fi;
      } else {
        ee[j] = sr;
      }
    }
    ee[m - 1] = 0.0;
  }
  __syncthreads();
  // V^T for the QL: Vt[c][r] = V[r][c] * phi[c]
  FOR2D(c, m, r, m) {  // coalesced writes of V^T
    const size_t e = (size_t)r * m + c;
    if (CPLX) {
      double tr, ti;
      cmul(Tr[e], Ti[e], wr[c], wi[c], tr, ti);
      Vr[(size_t)c * m + r] = tr;
      Vi[(size_t)c * m + r] = ti;
    } else {
      Vr[(size_t)c * m + r] = Tr[e];
    }
  }
  __syncthreads();

  RPROBE(3);
  if (a.method == 1) {
    // 5. implicit QL (reduced.py:117-172); rotations applied to columns of V
    const double epsm = 2.220446049250313e-16;
    for (int l = 0; l < m; ++l) {
      int sweeps = 0;
      while (true) {
        if (tid == 0) {
          int mm_ = l;
          while (mm_ < m - 1) {
            double dd = fabs(d[mm_]) + fabs(d[mm_ + 1]);
            if (fabs(ee[mm_]) <= epsm * dd) break;
            ++mm_;
          }
          int nrot = 0;
          if (mm_ != l) {
            ++sweeps;
            if (sweeps > 30) {
              nrot = -1;
            } else {
              double g = (d[l + 1] - d[l]) / (2.0 * ee[l]);
              double r = hypot(g, 1.0);
              g = d[mm_] - d[l] + ee[l] / (g + (g >= 0 ? r : -r));
              double s = 1.0, c = 1.0, p = 0.0;
              bool broke = false;
              for (int i = mm_ - 1; i >= l; --i) {
                double f = s * ee[i];
                double b = c * ee[i];
                // r = hypot(f, g), s = f / r, c = g / r with one reciprocal square
                // root on the serial critical path (values are O(1) here)
                const double q = fma(f, f, g * g);
                if (q == 0.0) {
                  ee[i + 1] = 0.0;
                  d[i + 1] -= p;
                  ee[mm_] = 0.0;
                  broke = true;
                  break;
                }
                const double ir = rsqrt(q);
                r = q * ir;
                ee[i + 1] = r;
                s = f * ir;
                c = g * ir;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * b;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - b;
                rc[i] = c;
                rs[i] = s;
                ++nrot;
              }
              if (!broke) {
                d[l] -= p;
                ee[l] = g;
                ee[mm_] = 0.0;
              }
            }
          }
          s_int[0] = (mm_ == l) ? 1 : 0;
          s_int[1] = nrot;
          s_int[2] = mm_;
        }
        __syncthreads();
        const int done = s_int[0], nrot = s_int[1], first = s_int[2];
        __syncthreads();
        if (nrot < 0) {
          if (tid == 0) *a.status = -1;
          return;
        }
        // rotation t acts on rows (i, i+1), i = first-1-t; the new row i is the
        // "row i+1" of rotation t+1, so it is carried in a register and only the
        // independent loads of row i go to memory.
        if (nrot > 0) {
          for (int r = tid; r < m; r += RT) {
            double cr = Vr[(size_t)first * m + r];
            double ci = CPLX ? Vi[(size_t)first * m + r] : 0.0;
            for (int t = 0; t < nrot; ++t) {
              const int i = first - 1 - t;
              const double c = rc[i], s = rs[i];
              const double zr = Vr[(size_t)i * m + r];
              Vr[(size_t)(i + 1) * m + r] = s * zr + c * cr;
              cr = c * zr - s * cr;
              if (CPLX) {
                const double zi = Vi[(size_t)i * m + r];
                Vi[(size_t)(i + 1) * m + r] = s * zi + c * ci;
                ci = c * zi - s * ci;
              }
            }
            const int last = first - nrot;
            Vr[(size_t)last * m + r] = cr;
            if (CPLX) Vi[(size_t)last * m + r] = ci;
          }
        }
        __syncthreads();
        if (done) break;
      }
    }

    // 6. stable ascending order, eps, Phi = L^-H V[:, order]
    int* order = reinterpret_cast<int*>(ur);
    for (int i = tid; i < m; i += RT) {
      double di = d[i];
      int rank = 0;
      for (int j = 0; j < m; ++j) {
        double dj = d[j];
        rank += (dj < di) || (dj == di && j < i);
      }
      a.eps[rank] = di;
      order[rank] = i;
    }
    __syncthreads();
    // X[i][c] = V[i][order[c]] = Vt[order[c]][i], into phi directly
    FOR2D(c, m, i, m) {
      const int oc = order[c];
      a.phre[(size_t)i * a.ldphi + c] = Vr[(size_t)oc * m + i];
      if (CPLX) a.phim[(size_t)i * a.ldphi + c] = Vi[(size_t)oc * m + i];
    }
    __syncthreads();
  } else {
    // 5'. tridiagonal eigenpairs by bisection (one thread per eigenvalue, the
    //     k-th smallest, ascending by construction) and inverse iteration with
    //     re-orthogonalisation inside clusters (LAPACK dstebz/dstein scheme).
    tridiag_bisect_invit(m, d, ee, a.eps, Zt, Wk, sh);
    __syncthreads();
    // Y = V Z (V^T held in (Vr, Vi), Z^T in Zt), straight into phi
    FOR2D(k, m, r, m) {
      double sr = 0.0, si = 0.0;
      const double* zk = Zt + (size_t)k * m;
      for (int c = 0; c < m; ++c) {
        const double z = zk[c];
        sr += Vr[(size_t)c * m + r] * z;
        if (CPLX) si += Vi[(size_t)c * m + r] * z;
      }
      a.phre[(size_t)r * a.ldphi + k] = sr;
      if (CPLX) a.phim[(size_t)r * a.ldphi + k] = si;
    }
    __syncthreads();
  }
  RPROBE(4);
  // right-looking backward solve L^H X = Y
  for (int i = m - 1; i >= 0; --i) {
    const double dr = Lr[(size_t)i * m + i];
    for (int c = tid; c < m; c += RT) {
      a.phre[(size_t)i * a.ldphi + c] /= dr;
      if (CPLX) a.phim[(size_t)i * a.ldphi + c] /= dr;
    }
    __syncthreads();
    FOR2D(r, i, c, m) {
      // X[r] -= conj(L[i][r]) X[i]
      const double lr = Lr[(size_t)i * m + r], xr = a.phre[(size_t)i * a.ldphi + c];
      if (CPLX) {
        const double li = -Li[(size_t)i * m + r], xi = a.phim[(size_t)i * a.ldphi + c];
        a.phre[(size_t)r * a.ldphi + c] -= lr * xr - li * xi;
        a.phim[(size_t)r * a.ldphi + c] -= lr * xi + li * xr;
      } else {
        a.phre[(size_t)r * a.ldphi + c] -= lr * xr;
      }
    }
    __syncthreads();
  }
  RPROBE(5);
  if (tid == 0) *a.status = 0;
}

size_t smem_for(int m) { return sizeof(double) * (4 * (size_t)m + 40); }

}  // namespace

void reduced_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_reduced_prof, sizeof(unsigned long long) * 8);
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_reduced_prof, z, sizeof(z));
}

size_t reduced_scratch_bytes(int m) { return sizeof(double) * (15 * (size_t)m * m + 8 * (size_t)m + 64); }

template <bool C>
static cudaError_t run_reduced(const RArgs& a, cudaStream_t st) {
  size_t smem = smem_for(a.m);
  static DevOnce cfg;
  if (cfg.first()) cudaFuncSetAttribute(reduced_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  reduced_kernel<C><<<1, RT, smem, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

cudaError_t chol_check_launch(int m, const double* bre, const double* bim, long long ld, int* fail,
                              double* scratch, cudaStream_t st) {
  RArgs a{};
  a.m = m; a.are = bre; a.aim = bim; a.bre = bre; a.bim = bim; a.ld = ld;
  a.status = fail; a.ws = scratch; a.check_only = 1;
  return bim ? run_reduced<true>(a, st) : run_reduced<false>(a, st);
}

cudaError_t reduced_eig_launch(int m, const double* are, const double* aim, const double* bre,
                               const double* bim, long long ld, double* eps, double* phre,
                               double* phim, long long ldphi, int* status, double* scratch,
                               cudaStream_t st) {
  RArgs a{};
  a.m = m; a.are = are; a.aim = aim; a.bre = bre; a.bim = bim; a.ld = ld;
  a.eps = eps; a.phre = phre; a.phim = phim; a.ldphi = ldphi;
  a.status = status; a.ws = scratch; a.check_only = 0;
  static const int method = getenv("FB_REDUCED_QL") ? 1 : 0;
  a.method = method;
  return aim ? run_reduced<true>(a, st) : run_reduced<false>(a, st);
}

}  // namespace fb
