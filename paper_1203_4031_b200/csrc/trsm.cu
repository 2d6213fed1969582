// Fused multi-RHS triangular sweeps for the dense shifted solves (dense.py:53-88).
//
// One cooperative kernel per sweep replaces the 2*N/32 launches of a blocked
// TRSM.  Blocks of 32 rows are finalised in processing order b(0), b(1), ...
// (ascending for the L / U^H sweeps, descending for U / L^H); at step t:
//   * "look-ahead" CTAs finalise the NEXT block for their 16-column chunk:
//       X_{b(t+1)} <- D_{b(t+1)} X_{b(t+1)} - G_{b(t+1)} X_{b(t)}
//     with D the diagonal-block inverse and G = D * M(b(t+1), b(t)) precomputed
//     per factor, so the critical path per step is ONE K=64 product;
//   * all CTAs stream the rank-32 update of the rows still pending,
//       X_i -= M(i, b(t)) X_{b(t)},   i in b(t+2) ...
//     as (32-row block, 16-column chunk) items, double-buffered with cp.async
//     (operator tile reused while consecutive items share a row block);
//   * one grid barrier per step (its gpu-scope fence also invalidates L1, so
//     the .ca cp.async reads of X never see stale lines).
// All products run on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA),
// complex as 4 real DMMAs on planar operands.
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
constexpr int PC = 18;   // C tile pitch
constexpr int A_SZ = 2 * BS * PA;
constexpr int B_SZ = 2 * BS * PB;
constexpr int C_SZ = 2 * BS * PC;
constexpr int STAGE = A_SZ + B_SZ + C_SZ;  // doubles per pipeline stage
constexpr int GM_BLK = 4 * BS * BS;        // per (variant, block): G re/im, D re/im

struct SweepArgs {
  int n, nrhs, nblk, variant;
  const double *lre, *lim;
  long long ld;
  const double* dinv;  // [nblk][L re, L im, U re, U im][32][32]
  const double* gmat;  // [4][nblk][G re, G im, D re, D im][32][32]
  double *xre, *xim;
  long long ldx;
  long long slu, sdinv, sx;  // batch strides (item b: + b * stride)
};

__device__ __forceinline__ void offset_item(SweepArgs& a, long long b) {
  a.lre += b * a.slu;
  a.lim += b * a.slu;
  a.dinv += b * a.sdinv;
  a.gmat += b * a.sdinv;
  a.xre += b * a.sx;
  a.xim += b * a.sx;
}

__device__ __forceinline__ int blk_at(const SweepArgs& a, int t) {
  return (a.variant == 0 || a.variant == 2) ? t : a.nblk - 1 - t;
}

// --- cp.async tile loaders ------------------------------------------------------
// A tile of M(i, b) (rows of block i, columns of block b); for the adjoint
// variants the tile is the transpose of LU(b, i) and is conjugated at use.
__device__ __forceinline__ void cp_m_tile(const SweepArgs& a, int bi, int bb, double* s) {
  const int i0 = bi * BS, b0 = bb * BS;
  const bool trans = a.variant >= 2;
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    int r, k;
    if (!trans) { r = e / BS; k = e % BS; } else { k = e / BS; r = e % BS; }
    const int gr = i0 + r, gk = b0 + k;
    const bool ok = gr < a.n && gk < a.n;
    const long long o = ok ? (trans ? (long long)gk * a.ld + gr : (long long)gr * a.ld + gk) : 0;
    cp_async8(s + r * PA + k, a.lre + o, ok);
    cp_async8(s + BS * PA + r * PA + k, a.lim + o, ok);
  }
}

// A tile from the per-factor operator store (G or D of this variant)
__device__ __forceinline__ void cp_op_tile(const double* src, double* s) {
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    const int r = e / BS, k = e % BS;
    cp_async8(s + r * PA + k, src + e, true);
    cp_async8(s + BS * PA + r * PA + k, src + BS * BS + e, true);
  }
}

// rows of block b, columns [c0, c0 + CW) of X into a tile with pitch P
template <int P>
__device__ __forceinline__ void cp_x_tile(const SweepArgs& a, int b, int c0, double* s) {
  const int r0 = b * BS;
  for (int e = threadIdx.x; e < BS * CW; e += TT) {
    const int k = e / CW, c = e % CW;
    const int gr = r0 + k, gc = c0 + c;
    const bool ok = gr < a.n && gc < a.nrhs;
    const long long o = ok ? (long long)gr * a.ldx + gc : 0;
    cp_async8(s + k * P + c, a.xre + o, ok);
    cp_async8(s + BS * P + k * P + c, a.xim + o, ok);
  }
}

// acc (8 rows x 16 cols per warp) += sign * A(32x32) B(32x16); conj_a negates Im(A)
__device__ __forceinline__ void tile_mma(double (&ar_)[2][2], double (&ai_)[2][2], const double* A,
                                         const double* B, double sign, double sign_i) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = w * 8 + (lane >> 2);
  const double* Ar = A;
  const double* Ai = A + BS * PA;
  const double* Br = B;
  const double* Bi = B + BS * PB;
#pragma unroll
  for (int k0 = 0; k0 < BS; k0 += 4) {
    const int k = k0 + (lane & 3);
    const double a_r = sign * Ar[row * PA + k];
    const double a_i = sign_i * Ai[row * PA + k];
    const double na_i = -a_i;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const double b_r = Br[k * PB + nt * 8 + (lane >> 2)];
      const double b_i = Bi[k * PB + nt * 8 + (lane >> 2)];
      dmma(ar_[nt][0], ar_[nt][1], a_r, b_r);
      dmma(ar_[nt][0], ar_[nt][1], na_i, b_i);
      dmma(ai_[nt][0], ai_[nt][1], a_r, b_i);
      dmma(ai_[nt][0], ai_[nt][1], a_i, b_r);
    }
  }
}

__device__ __forceinline__ void acc_from_smem(const double* C, double (&ar_)[2][2], double (&ai_)[2][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = w * 8 + (lane >> 2);
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = nt * 8 + 2 * (lane & 3) + e;
      ar_[nt][e] = C[r * PC + c];
      ai_[nt][e] = C[BS * PC + r * PC + c];
    }
}

__device__ __forceinline__ void acc_store(const SweepArgs& a, int b, int c0, const double (&ar_)[2][2],
                                          const double (&ai_)[2][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gr = b * BS + w * 8 + (lane >> 2);
  if (gr >= a.n) return;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int gc = c0 + nt * 8 + 2 * (lane & 3) + e;
      if (gc < a.nrhs) {
        const long long o = (long long)gr * a.ldx + gc;
        a.xre[o] = ar_[nt][e];
        a.xim[o] = ai_[nt][e];
      }
    }
}

__device__ __forceinline__ const double* op_ptr(const SweepArgs& a, int b, int which) {
  return a.gmat + ((size_t)a.variant * a.nblk + b) * GM_BLK + which * 2 * BS * BS;  // 0: G, 1: D
}

__global__ void __launch_bounds__(TT) sweep_kernel(SweepArgs a0) {
  extern __shared__ __align__(16) double s[];
  SweepArgs a = a0;
  offset_item(a, blockIdx.y);
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, g = blockIdx.x;
  const int C = ceil_div(a.nrhs, CW);
  const double conj_i = a.variant >= 2 ? -1.0 : 1.0;  // Im sign of the streamed M tiles
  double* st0 = s;
  double* st1 = s + STAGE;
  auto A_of = [&](double* st) { return st; };
  auto B_of = [&](double* st) { return st + A_SZ; };
  auto C_of = [&](double* st) { return st + A_SZ + B_SZ; };

  // prologue: the first block of the sweep is final after D
  {
    const int b0 = blk_at(a, 0);
    for (int c = g; c < C; c += G) {
      cp_op_tile(op_ptr(a, b0, 1), A_of(st0));
      cp_x_tile<PB>(a, b0, c * CW, B_of(st0));
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      double accr[2][2] = {{0, 0}, {0, 0}}, acci[2][2] = {{0, 0}, {0, 0}};
      tile_mma(accr, acci, A_of(st0), B_of(st0), 1.0, 1.0);
      acc_store(a, b0, c * CW, accr, acci);
      __syncthreads();
    }
  }
  grid.sync();

  for (int t = 0; t < a.nblk; ++t) {
    const int bt = blk_at(a, t);
    // look-ahead: finalise block b(t+1) = D X_{b(t+1)} - G X_{b(t)}
    if (t + 1 < a.nblk) {
      const int bn = blk_at(a, t + 1);
      for (int c = g; c < C; c += G) {
        cp_op_tile(op_ptr(a, bn, 1), A_of(st0));
        cp_x_tile<PB>(a, bn, c * CW, B_of(st0));
        cp_op_tile(op_ptr(a, bn, 0), A_of(st1));
        cp_x_tile<PB>(a, bt, c * CW, B_of(st1));
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        double accr[2][2] = {{0, 0}, {0, 0}}, acci[2][2] = {{0, 0}, {0, 0}};
        tile_mma(accr, acci, A_of(st0), B_of(st0), 1.0, 1.0);
        tile_mma(accr, acci, A_of(st1), B_of(st1), -1.0, -1.0);
        acc_store(a, bn, c * CW, accr, acci);
        __syncthreads();
      }
    }
    // streamed rank-32 updates, items (row block, chunk), contiguous per CTA
    const int nrest = a.nblk - t - 2;
    if (nrest > 0) {
      const int Q = nrest * C;
      int w = (g - C) % G;
      if (w < 0) w += G;
      const int qb = (int)((long long)w * Q / G), qe = (int)((long long)(w + 1) * Q / G);
      int a_rb[2] = {-1, -1};
      auto issue = [&](int q, int sidx) {
        double* st = sidx ? st1 : st0;
        const int rb = blk_at(a, t + 2 + q / C), c0 = (q % C) * CW;
        if (a_rb[sidx] != rb) {
          cp_m_tile(a, rb, bt, A_of(st));
          a_rb[sidx] = rb;
        }
        cp_x_tile<PB>(a, bt, c0, B_of(st));
        cp_x_tile<PC>(a, rb, c0, C_of(st));
        cp_async_commit();
      };
      if (qb < qe) issue(qb, 0);
      for (int q = qb; q < qe; ++q) {
        const int sidx = (q - qb) & 1;
        if (q + 1 < qe) {
          issue(q + 1, sidx ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        double* st = sidx ? st1 : st0;
        double accr[2][2], acci[2][2];
        acc_from_smem(C_of(st), accr, acci);
        tile_mma(accr, acci, A_of(st), B_of(st), -1.0, -conj_i);
        acc_store(a, blk_at(a, t + 2 + q / C), (q % C) * CW, accr, acci);
        __syncthreads();
      }
    }
    grid.sync();
  }
}

// Per (block, variant): D_v (the variant's diagonal inverse, conj-transposed for
// the adjoint sweeps) and G_v = D_v * M(b, prev(b)).
__global__ void __launch_bounds__(TT) gmat_kernel(SweepArgs a0) {
  __shared__ double Dr[BS * 33], Di[BS * 33], Mr[BS * 33], Mi[BS * 33];
  SweepArgs a = a0;
  offset_item(a, blockIdx.z);
  const int b = blockIdx.x, variant = blockIdx.y;
  const bool upper = variant == 1 || variant == 2;
  const bool trans = variant >= 2;
  const double* dr = a.dinv + (size_t)b * 4 * BS * BS + (upper ? 2 : 0) * BS * BS;
  const double* di = dr + BS * BS;
  double* out = const_cast<double*>(a.gmat) + ((size_t)variant * a.nblk + b) * GM_BLK;
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    const int r = e / BS, k = e % BS;
    const double vr = trans ? dr[k * BS + r] : dr[e];
    const double vi = trans ? -di[k * BS + r] : di[e];
    Dr[r * 33 + k] = vr;
    Di[r * 33 + k] = vi;
    out[2 * BS * BS + e] = vr;  // D
    out[3 * BS * BS + e] = vi;
  }
  const bool fwd = variant == 0 || variant == 2;
  const int prev = fwd ? b - 1 : b + 1;
  if (prev < 0 || prev >= a.nblk) {
    for (int e = threadIdx.x; e < BS * BS; e += TT) out[e] = out[BS * BS + e] = 0.0;
    return;
  }
  const int i0 = b * BS, p0 = prev * BS;
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    const int r = e / BS, k = e % BS;
    const int gr = i0 + r, gk = p0 + k;
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
    Mr[r * 33 + k] = vr;
    Mi[r * 33 + k] = vi;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BS * BS; e += TT) {
    const int r = e / BS, c = e % BS;
    double sr = 0.0, si = 0.0;
    for (int k = 0; k < BS; ++k) {
      const double xr = Dr[r * 33 + k], xi = Di[r * 33 + k];
      const double yr = Mr[k * 33 + c], yi = Mi[k * 33 + c];
      sr += xr * yr - xi * yi;
      si += xr * yi + xi * yr;
    }
    out[e] = sr;
    out[BS * BS + e] = si;
  }
}

int g_sweep_blocks = 0;

size_t sweep_smem() { return sizeof(double) * 2 * STAGE; }

}  // namespace

size_t gmat_doubles(int n) { return (size_t)4 * ceil_div(n, BS) * GM_BLK; }

cudaError_t gmat_launch(int n, int count, const double* lre, const double* lim, long long ld, long long slu,
                        const double* dinv, long long sdinv, double* gmat, cudaStream_t st) {
  SweepArgs a{};
  a.n = n; a.nblk = ceil_div(n, BS); a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.slu = slu; a.sdinv = sdinv; a.sx = 0;
  gmat_kernel<<<dim3(a.nblk, 4, count), TT, 0, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

cudaError_t sweep_launch(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                         long long ld, long long slu, const double* dinv, const double* gmat, long long sdinv,
                         double* xre, double* xim, long long ldx, long long sx, cudaStream_t st) {
  if (n <= 0 || nrhs <= 0 || count <= 0) return cudaSuccess;
  SweepArgs a{};
  a.n = n; a.nrhs = nrhs; a.nblk = ceil_div(n, BS); a.variant = variant;
  a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.xre = xre; a.xim = xim; a.ldx = ldx;
  a.slu = slu; a.sdinv = sdinv; a.sx = sx;
  size_t smem = sweep_smem();
  if (g_sweep_blocks == 0) {
    cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sweep_kernel, TT, smem);
    g_sweep_blocks = std::max(1, nb);
  }
  const int C = ceil_div(nrhs, CW);
  const long long items = (long long)std::max(0, a.nblk - 2) * C;
  const int cap = std::max(1, (g_sweep_blocks * kSMs) / count);
  if (cap < 1) return cudaErrorInvalidValue;
  int G = (int)std::min<long long>(cap, std::max<long long>(C, items));
  G = std::max(G, 1);
  void* args[] = {&a};
  count_launch();
  return cudaLaunchCooperativeKernel((void*)sweep_kernel, dim3(G, count), dim3(TT), args, smem, st);
}

}  // namespace fb
