// Banded backend (banded.py:50-178) — first, sequential-in-N restatement.
//
//   band_matvec   banded.py:50-65   y[j+s] += fb[kl+s, j] x[j], one thread per (row, rhs)
//   band_factor   banded.py:68-103  dgbtf2-style LU (kv = 2kl), one CTA walking the columns;
//                                   the shift z*FB - FA (banded.py:156-164) is formed on load
//   band_solve    banded.py:106-146 direct / adjoint, one thread per right-hand side with a
//                                   sliding window of the active rows in shared memory
//
// Working array: COLUMN-major, W[j*(3kl+1) + r] = ab[r, j] of the reference
// (r = kv + s holds the s-th subdiagonal of column j), planar complex.
#include "band.cuh"
#include "common.cuh"

namespace fb {

namespace {

__global__ void band_matvec_kernel(int n, int kl, int m, const double* __restrict__ fbr,
                                   const double* __restrict__ fbi, long long ldb,
                                   const double* __restrict__ xr, const double* __restrict__ xi,
                                   long long ldx, double* __restrict__ yr, double* __restrict__ yi,
                                   long long ldy) {
  long long total = (long long)n * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), c = (int)(e % m);
    double sr = 0.0, si = 0.0;
    for (int s = -kl; s <= kl; ++s) {  // y[i] += fb[kl+s, i-s] x[i-s]
      int j = i - s;
      if (j < 0 || j >= n) continue;
      double ar = fbr[(long long)(kl + s) * ldb + j];
      double ai = fbi ? fbi[(long long)(kl + s) * ldb + j] : 0.0;
      double br = xr[(long long)j * ldx + c];
      double bi = xi ? xi[(long long)j * ldx + c] : 0.0;
      sr += ar * br - ai * bi;
      si += ar * bi + ai * br;
    }
    yr[(long long)i * ldy + c] = sr;
    if (yi) yi[(long long)i * ldy + c] = si;
  }
}


// Tiled band matvec for kl <= 16: one CTA = RT consecutive rows x (32 * warps)
// columns.  The band entries of the CTA's rows are staged in shared memory
// row-aligned (sb[t][ii] = A(i0+ii, i0+ii-KL+t)) so every lane of a warp reads
// the same word (broadcast); each thread slides a register window of its
// column's x values (rows i-KL..i+KL) down the rows, so X is read from HBM
// once (plus a 2KL-row halo per tile) and Y written once.
constexpr int MV_RT = 128;
template <int KL, bool CPLX>
__global__ void __launch_bounds__(128) band_matvec_tiled(int n, int m, const double* __restrict__ fbr,
                                                         const double* __restrict__ fbi, long long ldb,
                                                         const double* __restrict__ xr,
                                                         const double* __restrict__ xi, long long ldx,
                                                         double* __restrict__ yr, double* __restrict__ yi,
                                                         long long ldy) {
  constexpr int W = 2 * KL + 1;
  extern __shared__ double sb[];  // [CPLX ? 2 : 1][W][MV_RT]
  const int i0 = blockIdx.x * MV_RT;
  const int rows = min(MV_RT, n - i0);
  for (int e = threadIdx.x; e < W * MV_RT; e += blockDim.x) {
    const int t = e / MV_RT, ii = e % MV_RT, i = i0 + ii, j = i - KL + t;
    double vr = 0.0, vi = 0.0;
    if (ii < rows && j >= 0 && j < n) {
      const long long o = (long long)(2 * KL - t) * ldb + j;  // fb[KL + (i - j)][j]
      vr = fbr[o];
      if (CPLX && fbi) vi = fbi[o];
    }
    sb[e] = vr;
    if (CPLX) sb[W * MV_RT + e] = vi;
  }
  __syncthreads();
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= m) return;
  auto ld = [&](int j, double& vr, double& vi) {
    vr = vi = 0.0;
    if (j >= 0 && j < n) {
      vr = xr[(long long)j * ldx + c];
      if (CPLX && xi) vi = xi[(long long)j * ldx + c];
    }
  };
  constexpr int QD = 8;  // rows prefetched ahead of the window (16: slower, 1.75 vs 1.58 ms at C4)
  double wr[W], wi[W], qr[QD], qi[QD];
#pragma unroll
  for (int t = 0; t < W; ++t) ld(i0 - KL + t, wr[t], wi[t]);
#pragma unroll
  for (int d = 0; d < QD; ++d) ld(i0 + KL + 1 + d, qr[d], qi[d]);
  for (int ii = 0; ii < rows; ++ii) {
    // numpy's order and rounding (banded.py:55-64): s = -KL..KL, i.e. j = i+KL
    // down to i-KL, each term a plain product added to y (no FMA contraction)
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int t = W - 1; t >= 0; --t) {
      const double ar = sb[t * MV_RT + ii];
      if (CPLX) {
        const double ai = sb[W * MV_RT + t * MV_RT + ii];
        sr = __dadd_rn(sr, __dsub_rn(__dmul_rn(ar, wr[t]), __dmul_rn(ai, wi[t])));
        si = __dadd_rn(si, __dadd_rn(__dmul_rn(ar, wi[t]), __dmul_rn(ai, wr[t])));
      } else {
        sr = __dadd_rn(sr, __dmul_rn(ar, wr[t]));
      }
    }
    const long long o = (long long)(i0 + ii) * ldy + c;
    yr[o] = sr;
    if (CPLX) yi[o] = si;
#pragma unroll
    for (int t = 0; t + 1 < W; ++t) {
      wr[t] = wr[t + 1];
      if (CPLX) wi[t] = wi[t + 1];
    }
    wr[W - 1] = qr[0];
    wi[W - 1] = qi[0];
#pragma unroll
    for (int d = 0; d + 1 < QD; ++d) {
      qr[d] = qr[d + 1];
      qi[d] = qi[d + 1];
    }
    ld(i0 + ii + KL + 1 + QD, qr[QD - 1], qi[QD - 1]);
  }
}

using MvFn = void (*)(int, int, const double*, const double*, long long, const double*, const double*, long long,
                      double*, double*, long long);
template <bool CPLX>
MvFn matvec_fn(int kl) {
  static const MvFn tbl[17] = {band_matvec_tiled<0, CPLX>,  band_matvec_tiled<1, CPLX>,  band_matvec_tiled<2, CPLX>,
                               band_matvec_tiled<3, CPLX>,  band_matvec_tiled<4, CPLX>,  band_matvec_tiled<5, CPLX>,
                               band_matvec_tiled<6, CPLX>,  band_matvec_tiled<7, CPLX>,  band_matvec_tiled<8, CPLX>,
                               band_matvec_tiled<9, CPLX>,  band_matvec_tiled<10, CPLX>, band_matvec_tiled<11, CPLX>,
                               band_matvec_tiled<12, CPLX>, band_matvec_tiled<13, CPLX>, band_matvec_tiled<14, CPLX>,
                               band_matvec_tiled<15, CPLX>, band_matvec_tiled<16, CPLX>};
  return tbl[kl];
}

// Shift into the working array: W[j][kl + r'] = z*FB[r'][j] - FA[r'][j], r' = 0..2kl.
__global__ void band_shift_kernel(int n, int kl, double zr, double zi, const double* __restrict__ far_,
                                  const double* __restrict__ fai, const double* __restrict__ fbr,
                                  const double* __restrict__ fbi, long long ldb, double* __restrict__ wr,
                                  double* __restrict__ wi) {
  const int W = 3 * kl + 1;
  long long total = (long long)n * W;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int j = (int)(e / W), r = (int)(e % W);
    double vr = 0.0, vi = 0.0;
    if (r >= kl) {
      int rr = r - kl;  // full-band row
      double ar = far_[(long long)rr * ldb + j], ai = fai ? fai[(long long)rr * ldb + j] : 0.0;
      double br, bi;
      if (fbr) {
        br = fbr[(long long)rr * ldb + j];
        bi = fbi ? fbi[(long long)rr * ldb + j] : 0.0;
      } else {
        br = (rr == kl) ? 1.0 : 0.0;
        bi = 0.0;
      }
      // numpy: shifted = zeros; shifted -= fa; shifted += z*fb  (banded.py:158-163)
      double pr = __dsub_rn(__dmul_rn(zr, br), __dmul_rn(zi, bi));
      double pi = __dadd_rn(__dmul_rn(zr, bi), __dmul_rn(zi, br));
      vr = (0.0 - ar) + pr;
      vi = (0.0 - ai) + pi;
      if (!fbr) {  // identity: shifted[kl, :] += z only on the diagonal row
        vr = (rr == kl) ? (0.0 - ar) + zr : (0.0 - ar);
        vi = (rr == kl) ? (0.0 - ai) + zi : (0.0 - ai);
      }
    }
    wr[(long long)j * W + r] = vr;
    wi[(long long)j * W + r] = vi;
  }
}

constexpr int FT = 256;

__global__ void __launch_bounds__(FT) band_factor_seq(int n, int kl, double* __restrict__ wr,
                                                      double* __restrict__ wi, int* __restrict__ ipiv,
                                                      int* __restrict__ info) {
  const int W = 3 * kl + 1, kv = 2 * kl, tid = threadIdx.x;
  __shared__ int s_jp, s_ju;
  __shared__ double s_l[2 * 128];
  int ju = 0;
  for (int j = 0; j < n; ++j) {
    const int km = min(kl, n - 1 - j);
    double* cr = wr + (long long)j * W;
    double* ci = wi + (long long)j * W;
    if (tid < 32) {
      double best = -1.0;
      int bi = 0;
      for (int i = tid; i <= km; i += 32) {
        double v = hypot(cr[kv + i], ci[kv + i]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (tid == 0) {
        int jp = bi;
        if (!(best > 0.0)) {
          atomicMin(info, j + 1);
          jp = 0;
        }
        ipiv[j] = j + jp;
        ju = max(ju, min(j + kl + jp, n - 1));
        s_jp = jp;
        s_ju = ju;
      }
    }
    __syncthreads();
    const int jp = s_jp;
    ju = s_ju;
    if (jp) {  // swap ab[kv+jp+j-c, c] <-> ab[kv+j-c, c], c = j..ju
      for (int c = j + tid; c <= ju; c += FT) {
        long long hi = (long long)c * W + kv + jp + j - c, lo = (long long)c * W + kv + j - c;
        double t = wr[hi]; wr[hi] = wr[lo]; wr[lo] = t;
        t = wi[hi]; wi[hi] = wi[lo]; wi[lo] = t;
      }
    }
    __syncthreads();
    const double pr = cr[kv], pim = ci[kv];
    const bool zero = !(pr != 0.0 || pim != 0.0);
    if (km > 0 && !zero) {
      const double den = pr * pr + pim * pim;
      const double ir = pr / den, ii = -pim / den;
      for (int i = tid; i < km; i += FT) {
        double xr = cr[kv + 1 + i], xi = ci[kv + 1 + i];
        double lr = xr * ir - xi * ii, li = xr * ii + xi * ir;
        cr[kv + 1 + i] = lr;
        ci[kv + 1 + i] = li;
        s_l[i] = lr;
        s_l[128 + i] = li;
      }
      __syncthreads();
      const int ncol = ju - j;
      for (int e = tid; e < ncol * km; e += FT) {
        int c = j + 1 + e / km, i = e % km;
        long long base = (long long)c * W + kv + j - c;
        double ur = wr[base], ui = wi[base];
        if (ur == 0.0 && ui == 0.0) continue;
        wr[base + 1 + i] -= s_l[i] * ur - s_l[128 + i] * ui;
        wi[base + 1 + i] -= s_l[i] * ui + s_l[128 + i] * ur;
      }
    }
    __syncthreads();
  }
}

// One thread per right-hand side column; window of rows [base, base + WN) in smem.
__global__ void band_solve_seq(int n, int kl, int nrhs, const double* __restrict__ wr,
                               const double* __restrict__ wi, const int* __restrict__ ipiv, int adjoint,
                               double* __restrict__ xr, double* __restrict__ xi, long long ldx) {
  extern __shared__ double win[];  // [WN][blockDim] re, then im
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int T = blockDim.x, t = threadIdx.x;
  const int W = 3 * kl + 1, kv = 2 * kl;
  const int WN = 2 * kl + 2;  // ring size
  double* wre = win;
  double* wim = win + WN * T;
  if (c >= nrhs) return;
  auto R = [&](int row) -> int { return ((row % WN) + WN) % WN * T + t; };
  auto load = [&](int row) {
    wre[R(row)] = xr[(long long)row * ldx + c];
    wim[R(row)] = xi[(long long)row * ldx + c];
  };
  auto store = [&](int row) {
    xr[(long long)row * ldx + c] = wre[R(row)];
    xi[(long long)row * ldx + c] = wim[R(row)];
  };
  if (!adjoint) {
    // forward: interleaved pivots + unit L (rows j..j+kl live)
    int hi = min(n, kl + 1);
    for (int r = 0; r < hi; ++r) load(r);
    for (int j = 0; j < n; ++j) {
      if (j + kl < n && j > 0) load(j + kl);  // rows up to j+kl resident
      if (kl > 0 && j < n - 1) {
        int p = ipiv[j];
        if (p != j) {
          double a = wre[R(j)], b = wim[R(j)];
          wre[R(j)] = wre[R(p)]; wim[R(j)] = wim[R(p)];
          wre[R(p)] = a; wim[R(p)] = b;
        }
        int km = min(kl, n - 1 - j);
        double x0r = wre[R(j)], x0i = wim[R(j)];
        const double* lr = wr + (long long)j * W + kv + 1;
        const double* li = wi + (long long)j * W + kv + 1;
        for (int i = 0; i < km; ++i) {
          double ar = lr[i], ai = li[i];
          wre[R(j + 1 + i)] -= ar * x0r - ai * x0i;
          wim[R(j + 1 + i)] -= ar * x0i + ai * x0r;
        }
      }
      store(j);
    }
    // backward: x[j] /= U[j,j]; x[j-lm..j-1] -= U[.., j] x[j]  (rows j-kv..j live)
    for (int r = n - 1; r >= max(0, n - 1 - kv); --r) load(r);
    for (int j = n - 1; j >= 0; --j) {
      if (j - kv >= 0 && j < n - 1) load(j - kv);
      double dr = wr[(long long)j * W + kv], di = wi[(long long)j * W + kv];
      double ar = wre[R(j)], ai = wim[R(j)];
      double den = dr * dr + di * di;
      double qr = (ar * dr + ai * di) / den, qi = (ai * dr - ar * di) / den;
      wre[R(j)] = qr;
      wim[R(j)] = qi;
      int lm = min(kv, j);
      const double* ur = wr + (long long)j * W + kv - lm;
      const double* ui = wi + (long long)j * W + kv - lm;
      for (int i = 0; i < lm; ++i) {
        double br = ur[i], bi = ui[i];
        wre[R(j - lm + i)] -= br * qr - bi * qi;
        wim[R(j - lm + i)] -= br * qi + bi * qr;
      }
      store(j);
    }
    return;
  }
  // adjoint: forward with U^H (needs rows j-kv..j), then L^H backward + reverse pivots
  for (int j = 0; j < n; ++j) {
    load(j);
    int lm = min(kv, j);
    double sr = wre[R(j)], si = wim[R(j)];
    const double* ur = wr + (long long)j * W + kv - lm;
    const double* ui = wi + (long long)j * W + kv - lm;
    for (int i = 0; i < lm; ++i) {  // x[j] -= conj(u) . x[j-lm+i]
      double br = ur[i], bi = -ui[i];
      double yr = wre[R(j - lm + i)], yi = wim[R(j - lm + i)];
      sr -= br * yr - bi * yi;
      si -= br * yi + bi * yr;
    }
    double dr = wr[(long long)j * W + kv], di = -wi[(long long)j * W + kv];
    double den = dr * dr + di * di;
    wre[R(j)] = (sr * dr + si * di) / den;
    wim[R(j)] = (si * dr - sr * di) / den;
    if (j - kv >= 0) store(j - kv);
  }
  for (int j = max(0, n - kv); j < n; ++j) store(j);
  if (kl > 0) {
    // rows j..j+kl live; walk down from n-2
    for (int r = n - 1; r >= max(0, n - 1 - kl); --r) load(r);
    for (int j = n - 2; j >= 0; --j) {
      if (j - 0 < n - 1 - kl) load(j);
      int km = min(kl, n - 1 - j);
      double sr = wre[R(j)], si = wim[R(j)];
      const double* lr = wr + (long long)j * W + kv + 1;
      const double* li = wi + (long long)j * W + kv + 1;
      for (int i = 0; i < km; ++i) {
        double ar = lr[i], ai = -li[i];
        double yr = wre[R(j + 1 + i)], yi = wim[R(j + 1 + i)];
        sr -= ar * yr - ai * yi;
        si -= ar * yi + ai * yr;
      }
      wre[R(j)] = sr;
      wim[R(j)] = si;
      int p = ipiv[j];
      if (p != j) {
        double a = wre[R(j)], b = wim[R(j)];
        wre[R(j)] = wre[R(p)]; wim[R(j)] = wim[R(p)];
        wre[R(p)] = a; wim[R(p)] = b;
      }
      if (j + kl + 1 <= n - 1) store(j + kl + 1);
    }
    for (int r = 0; r <= min(n - 1, kl); ++r) store(r);
  }
}

}  // namespace

cudaError_t band_matvec_launch(int n, int kl, int m, const double* fbr, const double* fbi, long long ldb,
                               const double* xr, const double* xi, long long ldx, double* yr, double* yi,
                               long long ldy, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  count_launch();
  const bool cplx = fbi != nullptr || xi != nullptr;
  if (kl >= 0 && kl <= 16 && (!cplx || yi != nullptr)) {
    const size_t smem = sizeof(double) * (cplx ? 2 : 1) * (2 * kl + 1) * MV_RT;
    const MvFn fn = cplx ? matvec_fn<true>(kl) : matvec_fn<false>(kl);
    static DevOnce cfg[2][17];
    if (cfg[cplx][kl].first()) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int nt = m >= 96 ? 96 : (m >= 64 ? 64 : 32);
    fn<<<dim3(ceil_div(n, MV_RT), ceil_div(m, nt)), nt, smem, st>>>(n, m, fbr, fbi, ldb, xr, xi, ldx, yr,
                                                                     cplx ? yi : nullptr, ldy);
    return cudaGetLastError();
  }
  long long total = (long long)n * m;
  int blocks = (int)std::min<long long>((total + 255) / 256, 16 * kSMs);
  band_matvec_kernel<<<blocks, 256, 0, st>>>(n, kl, m, fbr, fbi, ldb, xr, xi, ldx, yr, yi, ldy);
  return cudaGetLastError();
}

size_t band_fact_doubles(int n, int kl) { return (size_t)n * (3 * kl + 1); }

cudaError_t band_factor_launch(int n, int kl, double zr, double zi, const double* far_, const double* fai,
                               const double* fbr, const double* fbi, long long ldb, double* wr, double* wi,
                               int* ipiv, int* info, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (kl > 127) return cudaErrorInvalidValue;
  long long total = (long long)n * (3 * kl + 1);
  int blocks = (int)std::min<long long>((total + 255) / 256, 16 * kSMs);
  count_launch(2);
  band_shift_kernel<<<blocks, 256, 0, st>>>(n, kl, zr, zi, far_, fai, fbr, fbi, ldb, wr, wi);
  band_factor_seq<<<1, FT, 0, st>>>(n, kl, wr, wi, ipiv, info);
  return cudaGetLastError();
}

cudaError_t band_solve_launch(int n, int kl, int nrhs, const double* wr, const double* wi, const int* ipiv,
                              int adjoint, double* xr, double* xi, long long ldx, cudaStream_t st) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int T = 32;
  size_t smem = sizeof(double) * 2 * (2 * kl + 2) * T;
  count_launch();
  band_solve_seq<<<ceil_div(nrhs, T), T, smem, st>>>(n, kl, nrhs, wr, wi, ipiv, adjoint, xr, xi, ldx);
  return cudaGetLastError();
}

}  // namespace fb
