// Bandwidth-bound helpers of the FEAST refinement loop.
//
//   splitmix_fill   kernel.py:90-102 + 496-498 / 521-525 (bit-exact start block)
//   accumulate      kernel.py:108-124 (quadrature sum, numpy operation order)
//   symmetrize      kernel.py:380-381 (A_Q <- (A_Q + A_Q^H) / 2)
//   residuals       kernel.py:147-153 (column 1-norm ratios, +inf on zero denominator)
//   pack / unpack   numpy complex128 (interleaved) <-> planar device layout
#include <cstdint>

#include "common.cuh"
#include <algorithm>

#include "misc.cuh"

namespace fb {

namespace {

__device__ __forceinline__ double splitmix_u(unsigned long long seed, unsigned long long ctr) {
  unsigned long long z = seed + ctr * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return __dsub_rn(__dmul_rn((double)(z >> 11), 0x1p-52), 1.0);
}

// out(i, j) = u(seed, off + j*n + i)  (numpy reshape(order="F") of the stream)
__global__ void splitmix_kernel(unsigned long long seed, long long off_re, long long off_im, int n,
                                int m, double* __restrict__ re, double* __restrict__ im,
                                long long ld) {
  long long total = (long long)n * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    long long f = (long long)j * n + i;
    re[i * ld + j] = splitmix_u(seed, (unsigned long long)(off_re + f + 1));
    if (im) im[i * ld + j] = splitmix_u(seed, (unsigned long long)(off_im + f + 1));
  }
}

// mode 0: q -= h * (tr*xr - ti*xi)             (symmetric; h = w/2)
// mode 1: q -= (cr + i ci) * x                  (Hermitian direct / adjoint)
__global__ void accumulate_kernel(int mode, int n, int m, const double* __restrict__ xr,
                                  const double* __restrict__ xi, long long ldx,
                                  double* __restrict__ qr, double* __restrict__ qi, long long ldq,
                                  double h, double cr, double ci) {
  long long total = (long long)n * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    double a = xr[i * ldx + j], b = xi[i * ldx + j];
    if (mode == 0) {
      double v = __dsub_rn(__dmul_rn(cr, a), __dmul_rn(ci, b));
      qr[i * ldq + j] = __dsub_rn(qr[i * ldq + j], __dmul_rn(h, v));
    } else {
      double vr = __dsub_rn(__dmul_rn(cr, a), __dmul_rn(ci, b));
      double vi = __dadd_rn(__dmul_rn(cr, b), __dmul_rn(ci, a));
      qr[i * ldq + j] = __dsub_rn(qr[i * ldq + j], vr);
      qi[i * ldq + j] = __dsub_rn(qi[i * ldq + j], vi);
    }
  }
}

// All quadrature terms of one contour pass in one sweep over Q: each element
// of Q is read once, updated term by term in the caller's order with exactly
// accumulate_kernel's arithmetic (so the result equals the sequence of
// per-point accumulations bit for bit), and written once.
// V elements per thread (V = 2: 16-byte loads/stores when every row start is
// 16-byte aligned); the X loads of four terms are issued together before
// their (in-order) arithmetic, so each thread keeps 4 * 2 * V loads in flight.
template <int V>
__global__ void accumulate_terms_kernel(AccTerms t, int n, int m, long long ldx, double* __restrict__ qr,
                                        double* __restrict__ qi, long long ldq) {
  const int mv = m / V;
  const long long total = (long long)n * mv;
  const bool cplx = t.mode[0] != 0 && qi;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / mv), j = (int)(e % mv) * V;
    const long long ox = i * ldx + j, oq = i * ldq + j;
    double q_r[V], q_i[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      q_r[v] = qr[oq + v];
      q_i[v] = cplx ? qi[oq + v] : 0.0;
    }
    for (int k0 = 0; k0 < t.count; k0 += 4) {
      double a[4][V], b[4][V];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < t.count) {
          if (V == 2) {
            const double2 va = __ldcs(reinterpret_cast<const double2*>(t.xr[k0 + u] + ox));
            const double2 vb = __ldcs(reinterpret_cast<const double2*>(t.xi[k0 + u] + ox));
            a[u][0] = va.x; a[u][V - 1] = va.y;
            b[u][0] = vb.x; b[u][V - 1] = vb.y;
          } else {
            a[u][0] = __ldcs(t.xr[k0 + u] + ox);
            b[u][0] = __ldcs(t.xi[k0 + u] + ox);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u;
        if (k >= t.count) break;
        const double cr = t.cr[k], ci = t.ci[k];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (t.mode[k] == 0) {
            const double x = __dsub_rn(__dmul_rn(cr, a[u][v]), __dmul_rn(ci, b[u][v]));
            q_r[v] = __dsub_rn(q_r[v], __dmul_rn(t.h[k], x));
          } else {
            const double vr = __dsub_rn(__dmul_rn(cr, a[u][v]), __dmul_rn(ci, b[u][v]));
            const double vi = __dadd_rn(__dmul_rn(cr, b[u][v]), __dmul_rn(ci, a[u][v]));
            q_r[v] = __dsub_rn(q_r[v], vr);
            q_i[v] = __dsub_rn(q_i[v], vi);
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      qr[oq + v] = q_r[v];
      if (cplx) qi[oq + v] = q_i[v];
    }
  }
}

__global__ void symmetrize_kernel(int m, double* __restrict__ re, double* __restrict__ im,
                                  long long ld) {
  long long total = (long long)m * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    if (j < i) continue;
    double ar = re[i * ld + j], br = re[j * ld + i];
    double ai = im ? im[i * ld + j] : 0.0, bi = im ? im[j * ld + i] : 0.0;
    double nr = 0.5 * (ar + br);
    double ni = 0.5 * (ai - bi);
    re[i * ld + j] = nr;
    re[j * ld + i] = nr;
    if (im) {
      im[i * ld + j] = ni;
      if (j != i) im[j * ld + i] = -ni;
    }
  }
}

constexpr int RES_ROWS = 512;  // rows per partial-sum chunk

__global__ void residual_partial(int n, int m, const double* __restrict__ axr,
                                 const double* __restrict__ axi, const double* __restrict__ bxr,
                                 const double* __restrict__ bxi, long long ld,
                                 const double* __restrict__ lam, double scale,
                                 double* __restrict__ part) {
  const int chunk = blockIdx.x;
  const int r0 = chunk * RES_ROWS, r1 = min(n, r0 + RES_ROWS);
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double l = lam[j];
    double num = 0.0, den = 0.0;
    for (int i = r0; i < r1; ++i) {
      double br = bxr[i * ld + j], ar = axr[i * ld + j];
      if (axi) {
        double bi = bxi[i * ld + j], ai = axi[i * ld + j];
        num += hypot(ar - l * br, ai - l * bi);
        den += hypot(scale * br, scale * bi);
      } else {
        num += fabs(ar - l * br);
        den += fabs(scale * br);
      }
    }
    part[((size_t)chunk * m + j) * 2] = num;
    part[((size_t)chunk * m + j) * 2 + 1] = den;
  }
}

__global__ void residual_final(int chunks, int m, const double* __restrict__ part,
                               double* __restrict__ res) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double num = 0.0, den = 0.0;
  for (int c = 0; c < chunks; ++c) {
    num += part[((size_t)c * m + j) * 2];
    den += part[((size_t)c * m + j) * 2 + 1];
  }
  res[j] = den > 0.0 ? num / den : __longlong_as_double(0x7ff0000000000000ll);
}

// (num, den) per column without the division: the row-sharded residual of the
// multi-GPU path sums these over ranks first
__global__ void residual_sums(int chunks, int m, const double* __restrict__ part, double* __restrict__ sums) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double num = 0.0, den = 0.0;
  for (int c = 0; c < chunks; ++c) {
    num += part[((size_t)c * m + j) * 2];
    den += part[((size_t)c * m + j) * 2 + 1];
  }
  sums[2 * j] = num;
  sums[2 * j + 1] = den;
}

// interleaved complex (n x m, ld in complex elements) <-> planar (ldp)
__global__ void pack_kernel(int n, int m, const double* __restrict__ z, long long ldz,
                            double* __restrict__ re, double* __restrict__ im, long long ldp,
                            int to_planar) {
  long long total = (long long)n * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    if (to_planar) {
      double2 v = reinterpret_cast<const double2*>(z)[i * ldz + j];
      re[i * ldp + j] = v.x;
      if (im) im[i * ldp + j] = v.y;
    } else {
      double2 v;
      v.x = re[i * ldp + j];
      v.y = im ? im[i * ldp + j] : 0.0;
      reinterpret_cast<double2*>(const_cast<double*>(z))[i * ldz + j] = v;
    }
  }
}

int grid_for(long long total, int threads = 256) {
  long long b = (total + threads - 1) / threads;
  if (b > 16 * kSMs) b = 16 * kSMs;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t splitmix_launch(unsigned long long seed, long long off_re, long long off_im, int n, int m,
                            double* re, double* im, long long ld, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  count_launch();
  splitmix_kernel<<<grid_for((long long)n * m), 256, 0, st>>>(seed, off_re, off_im, n, m, re, im, ld);
  return cudaGetLastError();
}

cudaError_t accumulate_terms_launch(const AccTerms& t, int n, int m, long long ldx, double* qr, double* qi,
                                    long long ldq, cudaStream_t st) {
  if (n <= 0 || m <= 0 || t.count <= 0) return cudaSuccess;
  if (t.count > kMaxAccTerms) return cudaErrorInvalidValue;
  for (int k = 1; k < t.count; ++k)
    if ((t.mode[k] != 0) != (t.mode[0] != 0)) return cudaErrorInvalidValue;
  count_launch();
  bool vec = m % 2 == 0 && ldx % 2 == 0 && ldq % 2 == 0 &&
             ((reinterpret_cast<uintptr_t>(qr) | reinterpret_cast<uintptr_t>(qi)) & 15) == 0;
  for (int k = 0; k < t.count && vec; ++k)
    vec = ((reinterpret_cast<uintptr_t>(t.xr[k]) | reinterpret_cast<uintptr_t>(t.xi[k])) & 15) == 0;
  if (vec)
    accumulate_terms_kernel<2><<<grid_for((long long)n * m / 2), 256, 0, st>>>(t, n, m, ldx, qr, qi, ldq);
  else
    accumulate_terms_kernel<1><<<grid_for((long long)n * m), 256, 0, st>>>(t, n, m, ldx, qr, qi, ldq);
  return cudaGetLastError();
}

cudaError_t accumulate_launch(int mode, int n, int m, const double* xr, const double* xi,
                              long long ldx, double* qr, double* qi, long long ldq, double h,
                              double cr, double ci, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  count_launch();
  accumulate_kernel<<<grid_for((long long)n * m), 256, 0, st>>>(mode, n, m, xr, xi, ldx, qr, qi, ldq,
                                                                h, cr, ci);
  return cudaGetLastError();
}

cudaError_t symmetrize_launch(int m, double* re, double* im, long long ld, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  count_launch();
  symmetrize_kernel<<<grid_for((long long)m * m), 256, 0, st>>>(m, re, im, ld);
  return cudaGetLastError();
}

size_t residual_scratch_bytes(int n, int m) {
  return sizeof(double) * 2 * (size_t)ceil_div(n, RES_ROWS) * m;
}

cudaError_t residual_launch(int n, int m, const double* axr, const double* axi, const double* bxr,
                            const double* bxi, long long ld, const double* lam, double scale,
                            double* res, double* scratch, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  int chunks = ceil_div(n, RES_ROWS);
  count_launch(2);
  residual_partial<<<chunks, 128, 0, st>>>(n, m, axr, axi, bxr, bxi, ld, lam, scale, scratch);
  residual_final<<<ceil_div(m, 128), 128, 0, st>>>(chunks, m, scratch, res);
  return cudaGetLastError();
}

cudaError_t residual_sums_launch(int n, int m, const double* axr, const double* axi, const double* bxr,
                                 const double* bxi, long long ld, const double* lam, double scale,
                                 double* sums, double* scratch, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  int chunks = ceil_div(std::max(n, 1), RES_ROWS);
  count_launch(2);
  residual_partial<<<chunks, 128, 0, st>>>(n, m, axr, axi, bxr, bxi, ld, lam, scale, scratch);
  residual_sums<<<ceil_div(m, 128), 128, 0, st>>>(chunks, m, scratch, sums);
  return cudaGetLastError();
}

cudaError_t pack_launch(int n, int m, const double* z, long long ldz, double* re, double* im,
                        long long ldp, int to_planar, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  count_launch();
  pack_kernel<<<grid_for((long long)n * m), 256, 0, st>>>(n, m, z, ldz, re, im, ldp, to_planar);
  return cudaGetLastError();
}

}  // namespace fb
