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
};

__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double& cr, double& ci) {
  cr = ar * br - ai * bi;
  ci = ar * bi + ai * br;
}

template <bool CPLX>
__global__ void __launch_bounds__(RT, 1) reduced_kernel(RArgs a) {
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
  extern __shared__ double shd[];
  double* d = shd;           // [m]
  double* ee = d + m;        // [m]
  double* rc = ee + m;       // rotation cosines [m]
  double* rs = rc + m;       // rotation sines [m]
  double* sh = rs + m;       // reduction scratch [40]
  __shared__ int s_int[4];
  __shared__ double s_val[2];

  // finiteness (reduced.py:203-204)
  if (!a.check_only) {
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
  }
  if (m == 1 && !a.check_only) {  // reduced.py:205-210
    if (tid == 0) {
      double b00 = a.bre[0];
      if (b00 <= 0) {
        *a.status = -2;
      } else {
        a.eps[0] = a.are[0] / b00;
        a.phre[0] = 1.0 / sqrt(b00);
        if (CPLX) a.phim[0] = 0.0;
        *a.status = 0;
      }
    }
    return;
  }

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
              r = hypot(f, g);
              ee[i + 1] = r;
              if (r == 0.0) {
                d[i + 1] -= p;
                ee[mm_] = 0.0;
                broke = true;
                break;
              }
              s = f / r;
              c = g / r;
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
  if (tid == 0) *a.status = 0;
}

size_t smem_for(int m) { return sizeof(double) * (4 * (size_t)m + 40); }

}  // namespace

size_t reduced_scratch_bytes(int m) { return sizeof(double) * (8 * (size_t)m * m + 6 * (size_t)m + 64); }

template <bool C>
static cudaError_t run_reduced(const RArgs& a, cudaStream_t st) {
  size_t smem = smem_for(a.m);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(reduced_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cfg = true;
  }
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
  return aim ? run_reduced<true>(a, st) : run_reduced<false>(a, st);
}

}  // namespace fb
