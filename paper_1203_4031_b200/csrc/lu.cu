// Dense shifted complex LU with partial pivoting and its multi-RHS solves.
//
// Restates feastlib's dense backend (dense.py:30-88, _DenseOps dense.py:91-117)
// as a blocked algorithm for sm_100a:
//   * shift formation S = z B - A (dense.py:97-103), planar complex;
//   * right-looking blocked LU, outer block NB = 128 (trailing update is one
//     DMMA ZGEMM with K = 128), inner sub-panels of PW = 32 columns;
//   * each sub-panel is factored by ONE cooperative kernel that keeps the
//     panel rows resident in shared memory across all CTAs and exchanges a
//     single (|pivot|, row, row-data) record per CTA per column through L2
//     with one grid barrier per column: argmax pivot (first index on ties,
//     as np.argmax, dense.py:41), full-row swap, scaling and rank-1 update;
//   * the same kernel emits the inverses of the 32x32 unit-lower and upper
//     diagonal blocks, so every triangular solve downstream (the U12 block
//     row and the forward/backward solves of dense.py:53-88) is a DMMA GEMM;
//   * pivot vector semantics match lu_factor: piv[k] = row swapped with k at
//     step k (0-based), and an exactly zero pivot reports column k (the
//     SingularMatrixError of dense.py:42-43).
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm.cuh"
#include "lu.cuh"

namespace cg = cooperative_groups;

namespace fb {

namespace {

constexpr int PW = 32;         // sub-panel width (= diagonal block size of dinv)
constexpr int NB = 128;        // outer block (trailing-update K)
constexpr int PT = 128;        // threads per panel CTA
constexpr int SP = PW + 1;     // smem pitch of panel rows (conflict-free per-row access)

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
// Row interchanges piv[k0..k1) applied in order (reverse when rev) to
// columns [c0, c1) of a planar row-major matrix.  One thread per column.
// ---------------------------------------------------------------------------
__global__ void laswp_kernel(double* __restrict__ re, double* __restrict__ im, long long ld,
                             int c0, int c1, const int* __restrict__ piv, int k0, int k1, int rev) {
  int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  if (!rev) {
    for (int k = k0; k < k1; ++k) {
      int p = piv[k];
      if (p != k) {
        double t = re[(long long)k * ld + c];
        re[(long long)k * ld + c] = re[(long long)p * ld + c];
        re[(long long)p * ld + c] = t;
        if (im) {
          t = im[(long long)k * ld + c];
          im[(long long)k * ld + c] = im[(long long)p * ld + c];
          im[(long long)p * ld + c] = t;
        }
      }
    }
  } else {
    for (int k = k1 - 1; k >= k0; --k) {
      int p = piv[k];
      if (p != k) {
        double t = re[(long long)k * ld + c];
        re[(long long)k * ld + c] = re[(long long)p * ld + c];
        re[(long long)p * ld + c] = t;
        if (im) {
          t = im[(long long)k * ld + c];
          im[(long long)k * ld + c] = im[(long long)p * ld + c];
          im[(long long)p * ld + c] = t;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Cooperative sub-panel factorization.
// ---------------------------------------------------------------------------
struct PanelArgs {
  double* re;
  double* im;
  long long ld;
  int n, c0, pw, rpc;
  int* piv;
  int* info;
  double* xval;   // [2][G]
  int* xrow;      // [2][G]
  double* xdata;  // [2][G][2*PW]
  double* xrowr;  // [2][2*PW]
  double* linv;   // [2 planes][PW][PW] inverse of unit-lower diagonal block
  double* uinv;   // [2 planes][PW][PW] inverse of upper diagonal block
};

struct Best {
  double v;
  int r;
};
__device__ __forceinline__ Best better(Best a, Best b) {
  if (b.v > a.v || (b.v == a.v && b.r < a.r)) return b;
  return a;
}
__device__ __forceinline__ Best warp_best(Best b) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Best t;
    t.v = __shfl_xor_sync(0xffffffffu, b.v, o);
    t.r = __shfl_xor_sync(0xffffffffu, b.r, o);
    b = better(b, t);
  }
  return b;
}

__device__ Best block_best(Best b, Best* red) {
  b = warp_best(b);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = b;
  __syncthreads();
  if (threadIdx.x < 32) {
    Best t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : Best{-1.0, 0x7fffffff};
    t = warp_best(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

__global__ void __launch_bounds__(PT) panel_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int rows = a.n - a.c0;
  const int rbeg = a.c0 + g * a.rpc;
  const int rend = min(a.n, rbeg + a.rpc);
  const int cnt = max(0, rend - rbeg);
  double* sre = sm;                       // [rpc][SP]
  double* sim = sm + a.rpc * SP;          // [rpc][SP]
  double* prow = sim + a.rpc * SP;        // [2*PW] pivot row
  double* rrow = prow + 2 * PW;           // [2*PW] old row rj
  __shared__ Best red[PT / 32];
  __shared__ int s_gw;
  cg::grid_group grid = cg::this_grid();
  (void)rows;

  // load panel rows (columns c0 .. c0+pw) into shared memory
  for (int e = tid; e < cnt * PW; e += PT) {
    int lr = e / PW, c = e % PW;
    long long off = (long long)(rbeg + lr) * a.ld + a.c0 + c;
    bool ok = c < a.pw;
    sre[lr * SP + c] = ok ? a.re[off] : 0.0;
    sim[lr * SP + c] = ok ? a.im[off] : 0.0;
  }
  __syncthreads();

  for (int j = 0; j < a.pw; ++j) {
    const int rj = a.c0 + j;
    const int par = j & 1;
    // 1. local argmax of |a[r, j]| over own rows r >= rj
    Best b{-1.0, 0x7fffffff};
    for (int lr = tid; lr < cnt; lr += PT) {
      int gr = rbeg + lr;
      if (gr >= rj) {
        Best t{cabs_(sre[lr * SP + j], sim[lr * SP + j]), gr};
        b = better(b, t);
      }
    }
    b = block_best(b, red);
    // 2. publish (value, row, row data) and, for the owner, the old row rj
    if (tid == 0) {
      __stcg(a.xval + par * G + g, b.v);
      __stcg(a.xrow + par * G + g, b.r);
    }
    if (b.v >= 0.0 && b.r >= rbeg && b.r < rend) {
      int lr = b.r - rbeg;
      for (int c = tid; c < PW; c += PT) {
        __stcg(a.xdata + ((size_t)par * G + g) * 2 * PW + c, sre[lr * SP + c]);
        __stcg(a.xdata + ((size_t)par * G + g) * 2 * PW + PW + c, sim[lr * SP + c]);
      }
    }
    if (rj >= rbeg && rj < rend) {
      int lr = rj - rbeg;
      for (int c = tid; c < PW; c += PT) {
        __stcg(a.xrowr + par * 2 * PW + c, sre[lr * SP + c]);
        __stcg(a.xrowr + par * 2 * PW + PW + c, sim[lr * SP + c]);
      }
    }
    if (G > 1) {
      __threadfence();
      grid.sync();
    } else {
      __syncthreads();
    }
    // 3. global winner
    Best w{-1.0, 0x7fffffff};
    int wg = 0;
    for (int q = tid; q < G; q += PT) {
      Best t{__ldcg(a.xval + par * G + q), __ldcg(a.xrow + par * G + q)};
      Best nb = better(w, t);
      if (nb.r != w.r || nb.v != w.v) wg = q;
      w = nb;
    }
    Best wb = block_best(w, red);
    if (w.v == wb.v && w.r == wb.r && w.v >= 0.0) s_gw = wg;  // unique row -> unique writer
    for (int c = tid; c < 2 * PW; c += PT) rrow[c] = __ldcg(a.xrowr + par * 2 * PW + c);
    __syncthreads();
    const int gw = s_gw;
    for (int c = tid; c < 2 * PW; c += PT)
      prow[c] = __ldcg(a.xdata + ((size_t)par * G + gw) * 2 * PW + c);
    int p = wb.r;
    const bool zero = !(wb.v > 0.0);
    if (zero) {
      p = rj;
      if (g == 0 && tid == 0) atomicMin(a.info, rj + 1);
    }
    if (g == 0 && tid == 0) a.piv[rj] = p;
    __syncthreads();
    // 4. swap rows p <-> rj (full panel width), then scale and rank-1 update
    if (p != rj) {
      if (p >= rbeg && p < rend) {
        int lr = p - rbeg;
        for (int c = tid; c < PW; c += PT) {
          sre[lr * SP + c] = rrow[c];
          sim[lr * SP + c] = rrow[PW + c];
        }
      }
      if (rj >= rbeg && rj < rend) {
        int lr = rj - rbeg;
        for (int c = tid; c < PW; c += PT) {
          sre[lr * SP + c] = prow[c];
          sim[lr * SP + c] = prow[PW + c];
        }
      }
      __syncthreads();
    }
    if (!zero) {
      // reciprocal of the pivot
      double pr = prow[j], pi = prow[PW + j];
      double den = pr * pr + pi * pi;
      double ir = pr / den, ii = -pi / den;
      for (int lr = tid; lr < cnt; lr += PT) {
        int gr = rbeg + lr;
        if (gr <= rj) continue;
        double xr = sre[lr * SP + j], xi = sim[lr * SP + j];
        double lr_ = xr * ir - xi * ii, li = xr * ii + xi * ir;
        sre[lr * SP + j] = lr_;
        sim[lr * SP + j] = li;
        for (int c = j + 1; c < a.pw; ++c) {
          double ur = prow[c], ui = prow[PW + c];
          sre[lr * SP + c] -= lr_ * ur - li * ui;
          sim[lr * SP + c] -= lr_ * ui + li * ur;
        }
      }
    }
    __syncthreads();
  }

  // write back
  for (int e = tid; e < cnt * a.pw; e += PT) {
    int lr = e / a.pw, c = e % a.pw;
    long long off = (long long)(rbeg + lr) * a.ld + a.c0 + c;
    a.re[off] = sre[lr * SP + c];
    a.im[off] = sim[lr * SP + c];
  }
  // diagonal-block inverses (CTA 0 holds rows c0 .. c0+pw)
  if (g == 0 && tid < PW) {
    const int c = tid;
    double xr[PW], xi[PW];
    // unit-lower L: x = L^{-1} e_c
#pragma unroll
    for (int i = 0; i < PW; ++i) {
      double sr = (i == c) ? 1.0 : 0.0, si = 0.0;
      if (i < a.pw) {
#pragma unroll
        for (int k = 0; k < PW; ++k) {
          if (k < i) {
            double lr_ = sre[i * SP + k], li = sim[i * SP + k];
            sr -= lr_ * xr[k] - li * xi[k];
            si -= lr_ * xi[k] + li * xr[k];
          }
        }
      }
      xr[i] = sr;
      xi[i] = si;
    }
#pragma unroll
    for (int i = 0; i < PW; ++i) {
      a.linv[i * PW + c] = xr[i];
      a.linv[PW * PW + i * PW + c] = xi[i];
    }
    // upper U: x = U^{-1} e_c (identity padding beyond pw)
#pragma unroll
    for (int i = PW - 1; i >= 0; --i) {
      double sr = (i == c) ? 1.0 : 0.0, si = 0.0;
      if (i < a.pw) {
#pragma unroll
        for (int k = 0; k < PW; ++k) {
          if (k > i && k < a.pw) {
            double ur = sre[i * SP + k], ui = sim[i * SP + k];
            sr -= ur * xr[k] - ui * xi[k];
            si -= ur * xi[k] + ui * xr[k];
          }
        }
        double dr = sre[i * SP + i], di = sim[i * SP + i];
        double den = dr * dr + di * di;
        double qr = (sr * dr + si * di) / den, qi = (si * dr - sr * di) / den;
        sr = qr;
        si = qi;
      }
      xr[i] = sr;
      xi[i] = si;
    }
#pragma unroll
    for (int i = 0; i < PW; ++i) {
      a.uinv[i * PW + c] = xr[i];
      a.uinv[PW * PW + i * PW + c] = xi[i];
    }
  }
}

int g_panel_max_blocks = 0;  // co-resident panel CTAs per SM at max smem

}  // namespace

// Scratch needed by zgetrf beyond the factor itself.
size_t zgetrf_scratch_bytes(int n) {
  (void)n;
  const int Gmax = 4 * kSMs;
  return sizeof(double) * (2 * Gmax + 2 * (size_t)Gmax * 2 * PW + 2 * 2 * PW) +
         sizeof(int) * (2 * Gmax) + 256;
}

size_t dinv_doubles(int n) { return (size_t)ceil_div(n, PW) * 2 * 2 * PW * PW; }

cudaError_t shift_launch(int n, double zr, double zi, const double* are, const double* aim,
                         long long lda, const double* bre, const double* bim, long long ldb,
                         double* sre, double* sim, long long lds, cudaStream_t st) {
  long long total = (long long)n * n;
  int blocks = (int)std::min<long long>((total + 255) / 256, 8 * kSMs);
  shift_kernel<<<blocks, 256, 0, st>>>(n, zr, zi, are, aim, lda, bre, bim, ldb, sre, sim, lds);
  count_launch();
  return cudaGetLastError();
}

cudaError_t laswp_launch(double* re, double* im, long long ld, int c0, int c1, const int* piv,
                         int k0, int k1, int rev, cudaStream_t st) {
  if (c1 <= c0 || k1 <= k0) return cudaSuccess;
  int cols = c1 - c0;
  laswp_kernel<<<ceil_div(cols, 128), 128, 0, st>>>(re, im, ld, c0, c1, piv, k0, k1, rev);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t panel_launch(double* re, double* im, long long ld, int n, int c0, int pw, int* piv,
                                int* info, char* scratch, double* linv, double* uinv,
                                cudaStream_t st) {
  const int rows = n - c0;
  size_t smem_cap = 200 * 1024;
  int G = ceil_div(rows, 128);
  G = std::max(1, std::min(G, rows / PW));
  if (g_panel_max_blocks == 0) {
    cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap);
    int nb = 0;
    size_t probe = sizeof(double) * (2 * 128 * SP + 4 * PW);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, panel_kernel, PT, probe);
    g_panel_max_blocks = std::max(1, nb);
  }
  G = std::min(G, g_panel_max_blocks * kSMs);
  int rpc = ceil_div(rows, G);
  G = ceil_div(rows, rpc);
  size_t smem = sizeof(double) * (2 * (size_t)rpc * SP + 4 * PW);
  if (smem > smem_cap) return cudaErrorInvalidConfiguration;
  const int Gmax = 4 * kSMs;
  PanelArgs a;
  a.re = re; a.im = im; a.ld = ld; a.n = n; a.c0 = c0; a.pw = pw; a.rpc = rpc;
  a.piv = piv; a.info = info;
  double* d = reinterpret_cast<double*>(scratch);
  a.xval = d;
  a.xdata = d + 2 * Gmax;
  a.xrowr = a.xdata + 2 * (size_t)Gmax * 2 * PW;
  a.xrow = reinterpret_cast<int*>(a.xrowr + 2 * 2 * PW);
  a.linv = linv;
  a.uinv = uinv;
  void* args[] = {&a};
  count_launch();
  if (G > 1) {
    return cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(G), dim3(PT), args, smem, st);
  }
  panel_kernel<<<1, PT, smem, st>>>(a);
  return cudaGetLastError();
}

// In-place LU of the planar n x n matrix (re, im, ld).  piv[n] (device, 0-based),
// info (device int, pre-set by caller to INT_MAX: stays INT_MAX on success,
// else 1 + first zero-pivot column), dinv = dinv_doubles(n) doubles.
cudaError_t zgetrf(int n, double* re, double* im, long long ld, int* piv, int* info, double* dinv,
                   char* scratch, cudaStream_t st) {
  cudaError_t e;
  auto L = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW; };
  auto U = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW; };
  for (int k = 0; k < n; k += NB) {
    const int nb = std::min(NB, n - k);
    for (int s = 0; s < nb; s += PW) {
      const int c0 = k + s, pw = std::min(PW, nb - s), blk = c0 / PW;
      e = panel_launch(re, im, ld, n, c0, pw, piv, info, scratch, L(blk), U(blk), st);
      if (e != cudaSuccess) return e;
      // interchanges inside the outer block
      if ((e = laswp_launch(re, im, ld, k, c0, piv, c0, c0 + pw, 0, st))) return e;
      if ((e = laswp_launch(re, im, ld, c0 + pw, k + nb, piv, c0, c0 + pw, 0, st))) return e;
      const int rest = k + nb - (c0 + pw);
      if (rest > 0) {
        double* br = re + (long long)c0 * ld + c0 + pw;
        double* bi = im + (long long)c0 * ld + c0 + pw;
        // U row block: A[c0:c0+pw, c0+pw:k+nb] = Linv * A[...]  (in place, M=K=pw <= 64)
        e = gemm(1, pw, rest, pw, op_n(L(blk), L(blk) + PW * PW, PW), op_n(br, bi, ld), br, bi, ld,
                 1.0, 0.0, 0.0, 0.0, st);
        if (e) return e;
        const int below = n - (c0 + pw);
        if (below > 0) {
          e = gemm(1, below, rest, pw,
                   op_n(re + (long long)(c0 + pw) * ld + c0, im + (long long)(c0 + pw) * ld + c0, ld),
                   op_n(br, bi, ld), re + (long long)(c0 + pw) * ld + c0 + pw,
                   im + (long long)(c0 + pw) * ld + c0 + pw, ld, -1.0, 0.0, 1.0, 0.0, st);
          if (e) return e;
        }
      }
    }
    // interchanges outside the outer block
    if ((e = laswp_launch(re, im, ld, 0, k, piv, k, k + nb, 0, st))) return e;
    if ((e = laswp_launch(re, im, ld, k + nb, n, piv, k, k + nb, 0, st))) return e;
    const int right = n - (k + nb);
    if (right <= 0) continue;
    // U12 = L11^{-1} A12, by 32-row steps with the diagonal inverses
    for (int s = 0; s < nb; s += PW) {
      const int r0 = k + s, pw = std::min(PW, nb - s), blk = r0 / PW;
      double* xr = re + (long long)r0 * ld + k + nb;
      double* xi = im + (long long)r0 * ld + k + nb;
      e = gemm(1, pw, right, pw, op_n(L(blk), L(blk) + PW * PW, PW), op_n(xr, xi, ld), xr, xi, ld,
               1.0, 0.0, 0.0, 0.0, st);
      if (e) return e;
      const int rem = nb - s - pw;
      if (rem > 0) {
        e = gemm(1, rem, right, pw,
                 op_n(re + (long long)(r0 + pw) * ld + r0, im + (long long)(r0 + pw) * ld + r0, ld),
                 op_n(xr, xi, ld), re + (long long)(r0 + pw) * ld + k + nb,
                 im + (long long)(r0 + pw) * ld + k + nb, ld, -1.0, 0.0, 1.0, 0.0, st);
        if (e) return e;
      }
    }
    // trailing update A22 -= L21 U12 (K = nb)
    e = gemm(1, right, right, nb,
             op_n(re + (long long)(k + nb) * ld + k, im + (long long)(k + nb) * ld + k, ld),
             op_n(re + (long long)k * ld + k + nb, im + (long long)k * ld + k + nb, ld),
             re + (long long)(k + nb) * ld + k + nb, im + (long long)(k + nb) * ld + k + nb, ld, -1.0,
             0.0, 1.0, 0.0, st);
    if (e) return e;
  }
  return cudaSuccess;
}

// Solve op(A) X = B in place for X (n x nrhs planar, ldx) from zgetrf output.
// adjoint = 0: A X = B (dense.py:62-74); adjoint = 1: A^H X = B (dense.py:75-87).
cudaError_t zgetrs(int n, int nrhs, const double* re, const double* im, long long ld, const int* piv,
                   const double* dinv, int adjoint, double* xr, double* xi, long long ldx,
                   cudaStream_t st) {
  cudaError_t e;
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int nblk = ceil_div(n, PW);
  auto L = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW; };
  auto U = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW; };
  auto row = [&](const double* p, int r, int c) { return p + (long long)r * ld + c; };
  if (!adjoint) {
    if ((e = laswp_launch(xr, xi, ldx, 0, nrhs, piv, 0, n, 0, st))) return e;
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
  // A^H = U^H L^H P: forward with U^H, backward with L^H, then pivots reversed
  for (int b = 0; b < nblk; ++b) {
    const int r0 = b * PW, pw = std::min(PW, n - r0);
    double* x0r = xr + (long long)r0 * ldx;
    double* x0i = xi + (long long)r0 * ldx;
    if ((e = gemm(1, pw, nrhs, pw, op_c(U(b), U(b) + PW * PW, PW), op_n(x0r, x0i, ldx), x0r, x0i, ldx,
                  1.0, 0.0, 0.0, 0.0, st)))
      return e;
    const int below = n - r0 - pw;
    // X[below] -= (U[r0:r0+pw, below])^H X_b
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
    // X[0:r0] -= (L[r0:r0+pw, 0:r0])^H X_b
    if (r0 > 0 && (e = gemm(1, r0, nrhs, pw, op_c(row(re, r0, 0), row(im, r0, 0), ld),
                            op_n(x0r, x0i, ldx), xr, xi, ldx, -1.0, 0.0, 1.0, 0.0, st)))
      return e;
  }
  return laswp_launch(xr, xi, ldx, 0, nrhs, piv, 0, n, 1, st);
}

}  // namespace fb
