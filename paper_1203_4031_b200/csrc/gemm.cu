// FP64 / complex-FP64 GEMM on the sm_100a DMMA tensor pipe.
//
//   C(m x n) = alpha * op(A)(m x k) * op(B)(k x n) + beta * C
//
// Operands are described by (re, im, s0, s1, conj): op(A)(i, k) lives at
// re[i*s0 + k*s1] (+ i*im[...], conjugated when conj != 0).  That one
// descriptor covers N / T / C operands on row-major planar storage, which is
// every GEMM the FEAST hot path issues: the LU trailing update
// (A22 -= L21 U12), the blocked triangular-solve updates, A*Q / B*Q
// (kernel.py:372-376), the projections Q^H (AQ), Q^H (BQ) (kernel.py:377-379)
// and the Ritz products Q*Phi, AQ*Phi, BQ*Phi (kernel.py:411-413).
//
// Tiling: 64x64 CTA tile, 4 warps each owning a 32x32 block of 4x4 DMMA
// 8x8x4 tiles; operands stream global -> shared with cp.async in a 3-stage
// pipeline; shared layouts are chosen per operand contiguity so that both
// the cp.async stores and the fragment loads are bank-conflict free (64-bit
// elements have no ldmatrix path).  Complex products use 4 real DMMAs
// (re*re - im*im, re*im + im*re).  Split-K is deterministic: partial tiles go
// to a workspace and are reduced in a fixed order.
#include <cstdlib>

#include "common.cuh"
#include "gemm.cuh"

namespace fb {

namespace {

constexpr int BM = 64, BN = 64, BK = 8, STAGES = 4, THREADS = 128;
constexpr int PK = BK + 4;   // pitch of [row][k] layouts (12 doubles)
constexpr int PM = BM + 8;   // pitch of [k][row] layouts (72 doubles)

template <bool KC>
struct ATile {  // KC: k contiguous in global -> smem [BM][PK]; else [BK][PM]
  static constexpr int kElems = KC ? BM * PK : BK * PM;
  __device__ static int idx(int i, int k) { return KC ? i * PK + k : k * PM + i; }
};

template <bool CPLX, bool AKC, bool BNC>
__global__ void __launch_bounds__(THREADS, 2) gemm_kernel(GemmParams p) {
  constexpr int PL = CPLX ? 2 : 1;
  constexpr int AE = ATile<AKC>::kElems;
  constexpr int BE = ATile<!BNC>::kElems;  // B^T viewed as an A tile: n<->m
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                         // [STAGES][PL][AE]
  double* Bs = smem + STAGES * PL * AE;      // [STAGES][PL][BE]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int bz = blockIdx.z / p.splits;  // batch item (strided batch)
  const int z = blockIdx.z % p.splits;   // split-K slice
  const int kbeg = z * p.kchunk;
  const int kend = min(p.k, kbeg + p.kchunk);
  const int nk = kend > kbeg ? ceil_div(kend - kbeg, BK) : 0;

  const double* are = p.a.re + bz * p.bsa;
  const double* aim = p.a.im ? p.a.im + bz * p.bsa : nullptr;
  const double* bre = p.b.re + bz * p.bsb;
  const double* bim = p.b.im ? p.b.im + bz * p.bsb : nullptr;
  double* cre = p.cre + bz * p.bsc;
  double* cim = p.cim ? p.cim + bz * p.bsc : nullptr;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kbeg + kt * BK;
    double* as = As + stage * PL * AE;
    double* bs = Bs + stage * PL * BE;
#pragma unroll
    for (int r = 0; r < (BM * BK) / THREADS; ++r) {
      int e = tid + r * THREADS;
      int i, k;
      if (AKC) { i = e / BK; k = e % BK; } else { i = e % BM; k = e / BM; }
      int gi = m0 + i, gk = k0 + k;
      bool ok = gi < p.m && gk < kend;
      long long off = ok ? (long long)gi * p.a.s0 + (long long)gk * p.a.s1 : 0;
      int s = ATile<AKC>::idx(i, k);
      cp_async8(as + s, are + off, ok);
      if (CPLX) cp_async8(as + AE + s, (aim ? aim : are) + off, ok && aim);
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / THREADS; ++r) {
      int e = tid + r * THREADS;
      int j, k;
      if (BNC) { j = e % BN; k = e / BN; } else { j = e / BK; k = e % BK; }
      int gj = n0 + j, gk = k0 + k;
      bool ok = gj < p.n && gk < kend;
      long long off = ok ? (long long)gk * p.b.s0 + (long long)gj * p.b.s1 : 0;
      int s = ATile<!BNC>::idx(j, k);
      cp_async8(bs + s, bre + off, ok);
      if (CPLX) cp_async8(bs + BE + s, (bim ? bim : bre) + off, ok && bim);
    }
  };

  double accr[4][4][2], acci[4][4][2];
  // C += -A*B (alpha = -1, beta = 1, no split-K: the LU / solve updates): the
  // products are negated through the A fragments and accumulated from zero;
  // the epilogue adds them to C with ONE rounding per element (accumulating
  // onto C directly would round every one of the k FMAs at |C|'s magnitude:
  // sqrt(k) times the error, tools/dmma_rounding.py).
  const bool cinit = p.splits == 1 && p.alpha_re == -1.0 && p.alpha_im == 0.0 && p.beta_re == 1.0 &&
                     p.beta_im == 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        accr[a][b][e] = acci[a][b][e] = 0.0;
      }
  const double sgn = cinit ? -1.0 : 1.0;
  const double sa = p.a.conj ? -sgn : sgn;  // sign of the A imaginary fragments
  const double sb = p.b.conj ? -1.0 : 1.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nk) load_stage((kt + STAGES - 1) % STAGES, kt + STAGES - 1);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * PL * AE;
    const double* bs = Bs + (kt % STAGES) * PL * BE;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      const int kk = k4 + (lane & 3);
      double ar[4], ai[4], nai[4], br[4], bi[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int sA = ATile<AKC>::idx(wm + t * 8 + (lane >> 2), kk);
        ar[t] = sgn * as[sA];
        int sB = ATile<!BNC>::idx(wn + t * 8 + (lane >> 2), kk);
        br[t] = bs[sB];
        if (CPLX) {
          ai[t] = sa * as[AE + sA];
          nai[t] = -ai[t];
          bi[t] = sb * bs[BE + sB];
        }
      }
      // all first products, then the dependent second ones: 32 independent
      // accumulator chains between two DMMAs on the same accumulator
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dmma(accr[a][b][0], accr[a][b][1], ar[a], br[b]);
          if (CPLX) dmma(acci[a][b][0], acci[a][b][1], ar[a], bi[b]);
        }
      if (CPLX) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            dmma(accr[a][b][0], accr[a][b][1], nai[a], bi[b]);
            dmma(acci[a][b][0], acci[a][b][1], ai[a], br[b]);
          }
      }
    }
  }
  cp_async_wait<0>();

  // Epilogue.
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int i = m0 + wm + a * 8 + (lane >> 2);
        int j = n0 + wn + b * 8 + 2 * (lane & 3) + e;
        if (i >= p.m || j >= p.n) continue;
        double vr = accr[a][b][e], vi = CPLX ? acci[a][b][e] : 0.0;
        if (cinit) {
          const long long c = (long long)i * p.cs0 + (long long)j * p.cs1;
          cre[c] += vr;
          if (CPLX && cim) cim[c] += vi;
          continue;
        }
        if (p.splits > 1) {
          size_t plane = (size_t)p.m * p.n;
          double* w = p.ws + (size_t)z * PL * plane;
          w[(size_t)i * p.n + j] = vr;
          if (CPLX) w[plane + (size_t)i * p.n + j] = vi;
          continue;
        }
        long long c = (long long)i * p.cs0 + (long long)j * p.cs1;
        double outr = p.alpha_re * vr - p.alpha_im * vi;
        double outi = p.alpha_re * vi + p.alpha_im * vr;
        if (p.beta_re != 0.0 || p.beta_im != 0.0) {
          double cr = cre[c], ci = (CPLX && cim) ? cim[c] : 0.0;
          outr += p.beta_re * cr - p.beta_im * ci;
          outi += p.beta_re * ci + p.beta_im * cr;
        }
        cre[c] = outr;
        if (CPLX && cim) cim[c] = outi;
      }
}

// Fast path for the dominant complex case (LU trailing / in-block updates,
// dense multiplies): A k-contiguous, B n-contiguous, C row-major, every base
// pointer and leading dimension 16-byte aligned, no conjugation, no split-K.
// Same tiling and fragment order as gemm_kernel, but each thread streams
// fixed 16-byte chunks (pointer increments instead of per-element 64-bit
// index math, half the cp.async count), sign handling is compile-time (sign
// flips are integer ops, off the FP64 pipe the DMMAs run on); MODE 1
// (C -= A*B) negates the A fragments and adds the product to C once in the
// epilogue (one rounding per element, as gemm_kernel).
__device__ __forceinline__ double dneg(double v) {
  return __longlong_as_double(__double_as_longlong(v) ^ 0x8000000000000000ull);
}

template <int MODE, int NT>
__global__ void __launch_bounds__(NT, 2) zgemm_fast_kernel(GemmParams p) {
  // NT = 128: 4 warps of 32x32 (2x2); NT = 256: 8 warps of 32x16 (2x4), half
  // the accumulator registers per thread and twice the warps per SM
  constexpr int NB_ = NT == 128 ? 4 : 2;  // 8-column DMMA tiles per warp
  constexpr int WN = NB_ * 8;
  constexpr int WCOLS = BN / WN;          // warps along n
  constexpr int AE = ATile<true>::kElems;   // [BM][PK]
  constexpr int BE = ATile<false>::kElems;  // [BK][PM]  (B^T viewed as an A tile, n<->m)
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                 // [STAGES][2][AE]
  double* Bs = smem + STAGES * 2 * AE;  // [STAGES][2][BE]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / WCOLS) * 32, wn = (warp % WCOLS) * WN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int bz = blockIdx.z;
  const int nk = ceil_div(p.k, BK);
  const long long lda = p.a.s0, ldb = p.b.s0;
  const double* are = p.a.re + bz * p.bsa;
  const double* aim = p.a.im + bz * p.bsa;
  const double* bre = p.b.re + bz * p.bsb;
  const double* bim = p.b.im + bz * p.bsb;
  double* cre = p.cre + bz * p.bsc;
  double* cim = p.cim + bz * p.bsc;
  // A: 64 rows x 8 k = 256 16-byte chunks per plane; B: 8 k x 64 cols = 256
  constexpr int CH = 256 / NT;  // chunks per thread per plane
  int a_row[CH], a_kc[CH], b_k[CH], b_col[CH];
  const double* ap[CH];
  const double* bp[CH];
#pragma unroll
  for (int r = 0; r < CH; ++r) {
    const int e = tid + r * NT;
    a_row[r] = e >> 2;
    a_kc[r] = (e & 3) * 2;
    ap[r] = are + (long long)(m0 + a_row[r]) * lda + a_kc[r];
    b_k[r] = e >> 5;
    b_col[r] = (e & 31) * 2;
    bp[r] = bre + (long long)b_k[r] * ldb + n0 + b_col[r];
  }
  const long long aoff = aim - are, boff = bim - bre;
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * 2 * AE;
    double* bs = Bs + stage * 2 * BE;
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int gk = k0 + a_kc[r];
      const int bytes = (m0 + a_row[r] < p.m) ? (gk + 1 < p.k ? 16 : (gk < p.k ? 8 : 0)) : 0;
      const double* src = bytes ? ap[r] + k0 : are;
      const int s_ = a_row[r] * PK + a_kc[r];
      cp_async16(as + s_, src, bytes);
      cp_async16(as + AE + s_, bytes ? src + aoff : are, bytes);
    }
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int gk = k0 + b_k[r], gj = n0 + b_col[r];
      const int bytes = gk < p.k ? (gj + 1 < p.n ? 16 : (gj < p.n ? 8 : 0)) : 0;
      const double* src = bytes ? bp[r] + (long long)k0 * ldb : bre;
      const int s_ = b_k[r] * PM + b_col[r];
      cp_async16(bs + s_, src, bytes);
      cp_async16(bs + BE + s_, bytes ? src + boff : bre, bytes);
    }
  };
  double accr[4][NB_][2], acci[4][NB_][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NB_; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        accr[a][b][e] = acci[a][b][e] = 0.0;
      }
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  if (MODE == 1) {
    // the epilogue's C += product reads C once: pull the tile's 64-byte row
    // segments into L2 now so those loads do not wait on HBM at the end
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < NB_; ++b) {
        const int i = m0 + wm + a * 8 + (lane >> 2);
        const int j = n0 + wn + b * 8 + 2 * (lane & 3);
        if ((lane & 3) == 0 && i < p.m && j < p.n) {
          const long long c = (long long)i * p.cs0 + j;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(cre + c));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(cim + c));
        }
      }
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nk) load_stage((kt + STAGES - 1) % STAGES, kt + STAGES - 1);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * 2 * AE;
    const double* bs = Bs + (kt % STAGES) * 2 * BE;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      const int kk = k4 + (lane & 3);
      double x[4], y[4], z[4], br[NB_], bi[NB_];
#pragma unroll
      for (int t = 0; t < NB_; ++t) {
        const int sB = kk * PM + wn + t * 8 + (lane >> 2);
        br[t] = bs[sB];
        bi[t] = bs[BE + sB];
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int sA = (wm + t * 8 + (lane >> 2)) * PK + kk;
        const double ar = as[sA], ai = as[AE + sA];
        if (MODE == 1) {  // -(A B): re += (-ar) br + ai bi, im += (-ar) bi + (-ai) br
          x[t] = dneg(ar);
          y[t] = ai;
          z[t] = dneg(ai);
        } else {          // A B: re += ar br + (-ai) bi, im += ar bi + ai br
          x[t] = ar;
          y[t] = dneg(ai);
          z[t] = ai;
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB_; ++b) {
          dmma(accr[a][b][0], accr[a][b][1], x[a], br[b]);
          dmma(acci[a][b][0], acci[a][b][1], x[a], bi[b]);
        }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB_; ++b) {
          dmma(accr[a][b][0], accr[a][b][1], y[a], bi[b]);
          dmma(acci[a][b][0], acci[a][b][1], z[a], br[b]);
        }
    }
  }
  cp_async_wait<0>();
  if (MODE == 1) {
    // C += product: the loads of a half tile are issued together before any add
    // or store (cre/cim may alias as far as the compiler knows, so a plain
    // "c += v" loop serialises 32 load-add-store round trips per thread), as
    // 16-byte accesses where the row pair is aligned
    const bool v16 = (p.cs0 & 1) == 0 && ((uintptr_t)cre & 15) == 0 && ((uintptr_t)cim & 15) == 0;
#pragma unroll
    for (int a0 = 0; a0 < 4; a0 += 2) {
      double2 lr[2][NB_], li[2][NB_];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < NB_; ++b) {
          const int i = m0 + wm + (a0 + a) * 8 + (lane >> 2);
          const int j = n0 + wn + b * 8 + 2 * (lane & 3);
          const long long c = (long long)i * p.cs0 + j;
          lr[a][b] = li[a][b] = make_double2(0.0, 0.0);
          if (i < p.m && j + 1 < p.n && v16) {
            lr[a][b] = *reinterpret_cast<const double2*>(cre + c);
            li[a][b] = *reinterpret_cast<const double2*>(cim + c);
          } else if (i < p.m) {
            if (j < p.n) { lr[a][b].x = cre[c]; li[a][b].x = cim[c]; }
            if (j + 1 < p.n) { lr[a][b].y = cre[c + 1]; li[a][b].y = cim[c + 1]; }
          }
        }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < NB_; ++b) {
          const int i = m0 + wm + (a0 + a) * 8 + (lane >> 2);
          const int j = n0 + wn + b * 8 + 2 * (lane & 3);
          const long long c = (long long)i * p.cs0 + j;
          const double2 orr = make_double2(lr[a][b].x + accr[a0 + a][b][0], lr[a][b].y + accr[a0 + a][b][1]);
          const double2 oi = make_double2(li[a][b].x + acci[a0 + a][b][0], li[a][b].y + acci[a0 + a][b][1]);
          if (i < p.m && j + 1 < p.n && v16) {
            *reinterpret_cast<double2*>(cre + c) = orr;
            *reinterpret_cast<double2*>(cim + c) = oi;
          } else if (i < p.m) {
            if (j < p.n) { cre[c] = orr.x; cim[c] = oi.x; }
            if (j + 1 < p.n) { cre[c + 1] = orr.y; cim[c + 1] = oi.y; }
          }
        }
    }
    return;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NB_; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = m0 + wm + a * 8 + (lane >> 2);
        const int j = n0 + wn + b * 8 + 2 * (lane & 3) + e;
        if (i >= p.m || j >= p.n) continue;
        const long long c = (long long)i * p.cs0 + j;
        const double vr = accr[a][b][e], vi = acci[a][b][e];
        double outr = p.alpha_re * vr - p.alpha_im * vi;
        double outi = p.alpha_re * vi + p.alpha_im * vr;
        if (p.beta_re != 0.0 || p.beta_im != 0.0) {
          const double cr = cre[c], ci = cim[c];
          outr += p.beta_re * cr - p.beta_im * ci;
          outi += p.beta_re * ci + p.beta_im * cr;
        }
        cre[c] = outr;
        cim[c] = outi;
      }
}

template <bool CPLX>
__global__ void splitk_reduce(GemmParams p) {
  const size_t plane = (size_t)p.m * p.n;
  constexpr int PL = CPLX ? 2 : 1;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < plane;
       e += (size_t)gridDim.x * blockDim.x) {
    double vr = 0.0, vi = 0.0;
    for (int z = 0; z < p.splits; ++z) {
      vr += p.ws[(size_t)z * PL * plane + e];
      if (CPLX) vi += p.ws[(size_t)z * PL * plane + plane + e];
    }
    int i = (int)(e / p.n), j = (int)(e % p.n);
    long long c = (long long)i * p.cs0 + (long long)j * p.cs1;
    double outr = p.alpha_re * vr - p.alpha_im * vi;
    double outi = p.alpha_re * vi + p.alpha_im * vr;
    if (p.beta_re != 0.0 || p.beta_im != 0.0) {
      double cr = p.cre[c], ci = (CPLX && p.cim) ? p.cim[c] : 0.0;
      outr += p.beta_re * cr - p.beta_im * ci;
      outi += p.beta_re * ci + p.beta_im * cr;
    }
    p.cre[c] = outr;
    if (CPLX && p.cim) p.cim[c] = outi;
  }
}

template <bool CPLX, bool AKC, bool BNC>
cudaError_t launch_t(const GemmParams& p, cudaStream_t st) {
  constexpr int PL = CPLX ? 2 : 1;
  size_t smem = sizeof(double) * STAGES * PL * (ATile<AKC>::kElems + ATile<!BNC>::kElems);
  auto kern = gemm_kernel<CPLX, AKC, BNC>;
  static DevOnce configured;  // attribute set once per instantiation and device
  if (configured.first()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(ceil_div(p.n, BN), ceil_div(p.m, BM), p.splits * p.batch);
  kern<<<grid, THREADS, smem, st>>>(p);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || p.splits <= 1) return e;
  size_t plane = (size_t)p.m * p.n;
  int blocks = (int)std::min<size_t>((plane + 255) / 256, 4 * 148);
  splitk_reduce<CPLX><<<blocks, 256, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

static bool al16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

bool fast_ok(const GemmParams& p) {
  if (p.splits != 1 || p.k <= 0 || p.a.conj || p.b.conj || !p.a.im || !p.b.im || !p.cim) return false;
  if (p.a.s1 != 1 || p.b.s1 != 1 || p.cs1 != 1) return false;
  if ((p.a.s0 | p.b.s0 | p.cs0 | p.bsa | p.bsb) & 1) return false;
  return al16(p.a.re) && al16(p.a.im) && al16(p.b.re) && al16(p.b.im);
}

cudaError_t launch_fast(const GemmParams& p, cudaStream_t st) {
  const size_t smem = sizeof(double) * STAGES * 2 * (ATile<true>::kElems + ATile<false>::kElems);
  const bool mode1 = p.alpha_re == -1.0 && p.alpha_im == 0.0 && p.beta_re == 1.0 && p.beta_im == 0.0;
  constexpr int nt = 256;
  auto kern = mode1 ? zgemm_fast_kernel<1, 256> : zgemm_fast_kernel<0, 256>;
  static DevOnce configured[2];
  if (configured[mode1].first()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(ceil_div(p.n, BN), ceil_div(p.m, BM), p.batch);
  kern<<<grid, nt, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

size_t gemm_workspace_bytes(int cplx, int m, int n, int splits) {
  if (splits <= 1) return 0;
  return sizeof(double) * (cplx ? 2 : 1) * (size_t)splits * m * n;
}

int gemm_pick_splits(int m, int n, int k) {
  long long tiles = (long long)ceil_div(m, BM) * ceil_div(n, BN);
  if (tiles >= 2 * kSMs || k < 512) return 1;
  long long want = (2 * kSMs + tiles - 1) / tiles;
  long long maxs = k / 256;
  long long s = want < maxs ? want : maxs;
  return s < 1 ? 1 : (int)s;
}

cudaError_t gemm_launch(int cplx, GemmParams p, cudaStream_t st) {
  if (p.m <= 0 || p.n <= 0 || p.batch <= 0) return cudaSuccess;
  if (p.splits < 1) p.splits = 1;
  if (p.batch > 1) p.splits = 1;  // split-K workspace is per call, not per batch item
  if (p.k <= 0) {
    // C = beta * C (alpha * 0)
    p.k = 0;
    p.kchunk = 0;
    p.splits = 1;
  } else {
    p.kchunk = ceil_div(ceil_div(p.k, p.splits), BK) * BK;
    p.splits = ceil_div(p.k, p.kchunk);
  }
  bool akc = p.a.s1 == 1 || p.a.s0 != 1;   // k-contiguous (or generic) A
  bool bnc = p.b.s1 == 1 || p.b.s0 != 1;   // n-contiguous (or generic) B
  if (cplx && fast_ok(p)) return launch_fast(p, st);
  if (cplx) {
    if (akc && bnc) return launch_t<true, true, true>(p, st);
    if (akc && !bnc) return launch_t<true, true, false>(p, st);
    if (!akc && bnc) return launch_t<true, false, true>(p, st);
    return launch_t<true, false, false>(p, st);
  }
  if (akc && bnc) return launch_t<false, true, true>(p, st);
  if (akc && !bnc) return launch_t<false, true, false>(p, st);
  if (!akc && bnc) return launch_t<false, false, true>(p, st);
  return launch_t<false, false, false>(p, st);
}

}  // namespace fb
