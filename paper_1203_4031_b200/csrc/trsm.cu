// Fused multi-RHS triangular sweeps for the dense shifted solves (dense.py:53-88).
//
// One cooperative kernel per sweep replaces the 2*N/32 launches of a blocked
// TRSM.  Blocks of 32 rows are finalised in processing order b(0), b(1), ...
// (ascending for the L / U^H sweeps, descending for U / L^H); at step t:
//   * "look-ahead" CTAs finalise the NEXT block for their 16-column chunk:
//       X_{b(t+1)} <- D_{b(t+1)} X_{b(t+1)} - G_{b(t+1)} X_{b(t)}
//     with D the diagonal-block inverse and G = D * M(b(t+1), b(t)) precomputed
//     per factor, so the critical path per step is ONE K=64 product;
//   * every other CTA streams the rank-32 update of the rows still pending,
//       X_i -= M(i, b(t)) X_{b(t)},   i in b(t+2) ...
//     with the 32x32 operator tile held in shared memory across all chunks;
//   * one grid barrier per step.
// All products run on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA),
// complex as 4 real DMMAs on planar operands.  X is always read with ld.cg
// (L2) because other CTAs rewrite it between barriers.
//
//   variant 0  L   forward  (direct solve, after the row gather P B)
//   variant 1  U   backward (direct solve)
//   variant 2  U^H forward  (adjoint solve)
//   variant 3  L^H backward (adjoint solve, then the row scatter P^T)
#include <cooperative_groups.h>

#include "common.cuh"
#include "trsm.cuh"

namespace cg = cooperative_groups;

namespace fb {

namespace {

constexpr int BS = 32;   // block rows (= PW of the factorization)
constexpr int CW = 16;   // right-hand-side columns per chunk
constexpr int TT = 128;  // threads (4 warps, 8 rows each)
constexpr int PA = 36;   // A tile pitch: conflict-free A fragments
constexpr int PB = 24;   // B tile pitch: conflict-free B fragments

struct SweepArgs {
  int n, nrhs, nblk, variant;
  const double *lre, *lim;
  long long ld;
  const double* dinv;   // [nblk][L re, L im, U re, U im][32][32]
  const double* gmat;   // [4][nblk][2][32][32]
  double *xre, *xim;
  long long ldx;
};

__device__ __forceinline__ int blk_at(const SweepArgs& a, int t) {
  return (a.variant == 0 || a.variant == 2) ? t : a.nblk - 1 - t;
}

// A tile (32 x 32 complex) of the operator M(i, b): rows of block i, columns of block b.
__device__ void load_m_tile(const SweepArgs& a, int bi, int bb, double* sr, double* si) {
  const int i0 = bi * BS, b0 = bb * BS;
  const bool trans = a.variant >= 2;
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    int r, k;
    if (!trans) { r = e / BS; k = e % BS; } else { k = e / BS; r = e % BS; }
    int gr = i0 + r, gk = b0 + k;
    double vr = 0.0, vi = 0.0;
    if (gr < a.n && gk < a.n) {
      if (!trans) {
        vr = a.lre[(long long)gr * a.ld + gk];
        vi = a.lim[(long long)gr * a.ld + gk];
      } else {
        vr = a.lre[(long long)gk * a.ld + gr];
        vi = -a.lim[(long long)gk * a.ld + gr];
      }
    }
    sr[r * PA + k] = vr;
    si[r * PA + k] = vi;
  }
}

// A tile of D_b (diagonal inverse for this variant)
__device__ void load_d_tile(const SweepArgs& a, int b, double* sr, double* si) {
  const double* base = a.dinv + (size_t)b * 4 * BS * BS;
  const bool upper = a.variant == 1 || a.variant == 2;
  const bool trans = a.variant >= 2;
  const double* pr = base + (upper ? 2 : 0) * BS * BS;
  const double* pi = pr + BS * BS;
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    int r = e / BS, k = e % BS;
    if (!trans) {
      sr[r * PA + k] = pr[r * BS + k];
      si[r * PA + k] = pi[r * BS + k];
    } else {
      sr[r * PA + k] = pr[k * BS + r];
      si[r * PA + k] = -pi[k * BS + r];
    }
  }
}

__device__ void load_g_tile(const SweepArgs& a, int b, double* sr, double* si) {
  const double* pr = a.gmat + ((size_t)a.variant * a.nblk + b) * 2 * BS * BS;
  const double* pi = pr + BS * BS;
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    int r = e / BS, k = e % BS;
    sr[r * PA + k] = pr[e];
    si[r * PA + k] = pi[e];
  }
}

// B tile: rows of block b, columns [c0, c0+CW) of X (zero outside)
__device__ void load_x_tile(const SweepArgs& a, int b, int c0, double* sr, double* si) {
  const int r0 = b * BS;
  for (int e = threadIdx.x; e < BS * CW; e += TT) {
    int k = e / CW, c = e % CW;
    int gr = r0 + k, gc = c0 + c;
    double vr = 0.0, vi = 0.0;
    if (gr < a.n && gc < a.nrhs) {
      vr = __ldcg(a.xre + (long long)gr * a.ldx + gc);
      vi = __ldcg(a.xim + (long long)gr * a.ldx + gc);
    }
    sr[k * PB + c] = vr;
    si[k * PB + c] = vi;
  }
}

// acc (8 rows x 16 cols per warp) += sign * A(32x32) B(32x16)
__device__ __forceinline__ void tile_mma(double (&ar_)[2][2], double (&ai_)[2][2], const double* Ar,
                                         const double* Ai, const double* Br, const double* Bi,
                                         double sign) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = w * 8 + (lane >> 2);
#pragma unroll
  for (int k0 = 0; k0 < BS; k0 += 4) {
    const int k = k0 + (lane & 3);
    double a_r = sign * Ar[row * PA + k];
    double a_i = sign * Ai[row * PA + k];
    double na_i = -a_i;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      double b_r = Br[k * PB + nt * 8 + (lane >> 2)];
      double b_i = Bi[k * PB + nt * 8 + (lane >> 2)];
      dmma(ar_[nt][0], ar_[nt][1], a_r, b_r);
      dmma(ar_[nt][0], ar_[nt][1], na_i, b_i);
      dmma(ai_[nt][0], ai_[nt][1], a_r, b_i);
      dmma(ai_[nt][0], ai_[nt][1], a_i, b_r);
    }
  }
}

__device__ __forceinline__ void acc_io(const SweepArgs& a, int b, int c0, double (&ar_)[2][2],
                                       double (&ai_)[2][2], bool store) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gr = b * BS + w * 8 + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int gc = c0 + nt * 8 + 2 * (lane & 3) + e;
      const bool ok = gr < a.n && gc < a.nrhs;
      const long long o = (long long)gr * a.ldx + gc;
      if (store) {
        if (ok) {
          a.xre[o] = ar_[nt][e];
          a.xim[o] = ai_[nt][e];
        }
      } else {
        ar_[nt][e] = ok ? __ldcg(a.xre + o) : 0.0;
        ai_[nt][e] = ok ? __ldcg(a.xim + o) : 0.0;
      }
    }
}

__device__ void finalize_first(const SweepArgs& a, int b, int c0, double* s) {
  double* Dr = s;
  double* Di = Dr + BS * PA;
  double* Br = Di + BS * PA;
  double* Bi = Br + BS * PB;
  __syncthreads();
  load_d_tile(a, b, Dr, Di);
  load_x_tile(a, b, c0, Br, Bi);
  __syncthreads();
  double accr[2][2] = {{0, 0}, {0, 0}}, acci[2][2] = {{0, 0}, {0, 0}};
  tile_mma(accr, acci, Dr, Di, Br, Bi, 1.0);
  acc_io(a, b, c0, accr, acci, true);
}

__global__ void __launch_bounds__(TT) sweep_kernel(SweepArgs a) {
  extern __shared__ __align__(16) double s[];
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, g = blockIdx.x;
  const int C = ceil_div(a.nrhs, CW);
  // smem: two A tiles (2 planes each) and two B tiles
  double* A1r = s;
  double* A1i = A1r + BS * PA;
  double* A2r = A1i + BS * PA;
  double* A2i = A2r + BS * PA;
  double* B1r = A2i + BS * PA;
  double* B1i = B1r + BS * PB;
  double* B2r = B1i + BS * PB;
  double* B2i = B2r + BS * PB;

  // prologue: the first block of the sweep is final after D
  for (int c = g; c < C; c += G) finalize_first(a, blk_at(a, 0), c * CW, s);
  grid.sync();

  for (int t = 0; t < a.nblk; ++t) {
    const int bt = blk_at(a, t);
    // look-ahead: finalise block b(t+1)
    if (t + 1 < a.nblk) {
      const int bn = blk_at(a, t + 1);
      for (int c = g; c < C; c += G) {
        __syncthreads();
        load_d_tile(a, bn, A1r, A1i);
        load_g_tile(a, bn, A2r, A2i);
        load_x_tile(a, bn, c * CW, B1r, B1i);
        load_x_tile(a, bt, c * CW, B2r, B2i);
        __syncthreads();
        double accr[2][2] = {{0, 0}, {0, 0}}, acci[2][2] = {{0, 0}, {0, 0}};
        tile_mma(accr, acci, A1r, A1i, B1r, B1i, 1.0);
        tile_mma(accr, acci, A2r, A2i, B2r, B2i, -1.0);
        acc_io(a, bn, c * CW, accr, acci, true);
      }
    }
    // streamed updates of the rows still pending
    const int nrest = a.nblk - t - 2;
    if (nrest > 0) {
      int q0 = (g - C) % G;
      if (q0 < 0) q0 += G;
      for (int q = q0; q < nrest; q += G) {
        const int bi = blk_at(a, t + 2 + q);
        __syncthreads();
        load_m_tile(a, bi, bt, A1r, A1i);
        for (int c = 0; c < C; ++c) {
          __syncthreads();
          load_x_tile(a, bt, c * CW, B1r, B1i);
          __syncthreads();
          double accr[2][2], acci[2][2];
          acc_io(a, bi, c * CW, accr, acci, false);
          tile_mma(accr, acci, A1r, A1i, B1r, B1i, -1.0);
          acc_io(a, bi, c * CW, accr, acci, true);
        }
      }
    }
    __threadfence();
    grid.sync();
  }
}

// G_b = D_b * M(b, prev(b)) for the four sweep variants (one CTA per (b, variant)).
__global__ void __launch_bounds__(TT) gmat_kernel(SweepArgs a) {
  extern __shared__ __align__(16) double s[];
  const int b = blockIdx.x, variant = blockIdx.y;
  SweepArgs v = a;
  v.variant = variant;
  double* Dr = s;
  double* Di = Dr + BS * PA;
  double* Mr = Di + BS * PA;
  double* Mi = Mr + BS * PA;
  const bool fwd = variant == 0 || variant == 2;
  const int prev = fwd ? b - 1 : b + 1;
  double* outr = const_cast<double*>(a.gmat) + ((size_t)variant * a.nblk + b) * 2 * BS * BS;
  double* outi = outr + BS * BS;
  if (prev < 0 || prev >= a.nblk) {
    for (int e = threadIdx.x; e < BS * BS; e += TT) outr[e] = outi[e] = 0.0;
    return;
  }
  load_d_tile(v, b, Dr, Di);
  load_m_tile(v, b, prev, Mr, Mi);
  __syncthreads();
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    int r = e / BS, c = e % BS;
    double sr = 0.0, si = 0.0;
    for (int k = 0; k < BS; ++k) {
      double xr = Dr[r * PA + k], xi = Di[r * PA + k];
      double yr = Mr[k * PA + c], yi = Mi[k * PA + c];
      sr += xr * yr - xi * yi;
      si += xr * yi + xi * yr;
    }
    outr[e] = sr;
    outi[e] = si;
  }
}

int g_sweep_blocks = 0;

size_t sweep_smem() { return sizeof(double) * (4 * BS * PA + 4 * BS * PB); }

}  // namespace

size_t gmat_doubles(int n) { return (size_t)4 * ceil_div(n, BS) * 2 * BS * BS; }

cudaError_t gmat_launch(int n, const double* lre, const double* lim, long long ld, const double* dinv,
                        double* gmat, cudaStream_t st) {
  SweepArgs a{};
  a.n = n; a.nblk = ceil_div(n, BS); a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  size_t smem = sizeof(double) * 4 * BS * PA;
  gmat_kernel<<<dim3(a.nblk, 4), TT, smem, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

cudaError_t sweep_launch(int variant, int n, int nrhs, const double* lre, const double* lim, long long ld,
                         const double* dinv, const double* gmat, double* xre, double* xim, long long ldx,
                         cudaStream_t st) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  SweepArgs a{};
  a.n = n; a.nrhs = nrhs; a.nblk = ceil_div(n, BS); a.variant = variant;
  a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.xre = xre; a.xim = xim; a.ldx = ldx;
  size_t smem = sweep_smem();
  if (g_sweep_blocks == 0) {
    cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sweep_kernel, TT, smem);
    g_sweep_blocks = std::max(1, nb);
  }
  const int C = ceil_div(nrhs, CW);
  int G = std::min(g_sweep_blocks * kSMs, std::max(C, C + a.nblk - 2));
  G = std::max(G, 1);
  void* args[] = {&a};
  count_launch();
  return cudaLaunchCooperativeKernel((void*)sweep_kernel, dim3(G), dim3(TT), args, smem, st);
}

}  // namespace fb
