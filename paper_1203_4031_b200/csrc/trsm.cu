// Fused multi-RHS triangular sweeps for the dense shifted solves (dense.py:53-88).
//
// One cooperative kernel per sweep replaces the 2*N/32 launches of a blocked
// TRSM.  Blocks of 32 rows are finalised in processing order b(0), b(1), ...
// (ascending for the L / U^H sweeps, descending for U / L^H).  The right-hand
// sides are cut into 32-column chunks and every CTA owns ONE chunk for the
// whole sweep (a group of S CTAs per chunk), so at step t it stages the final
// block X_{b(t)}[:, chunk] in shared memory once and then:
//   * sub-CTA 0 of the group finalises the NEXT block ("look-ahead"):
//       X_{b(t+1)} <- D_{b(t+1)} X_{b(t+1)} - G_{b(t+1)} X_{b(t)}
//     with D the diagonal-block inverse and G = D * M(b(t+1), b(t)) precomputed
//     per factor, so the critical path per step is ONE K=64 product;
//   * the group streams the rank-32 update of its share of the pending rows,
//       X_i -= M(i, b(t)) X_{b(t)},   i in b(t+2) ...
//     with the 32x32 M tiles double-buffered by 16-byte cp.async and the X_i
//     accumulators prefetched straight into registers (L2-only loads);
//   * no grid barriers: per (row block, chunk) counters in global memory
//     (release/acquire) let each CTA start a step as soon as the blocks it
//     reads are final, so steps overlap (see sweep_body).
// All products run on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA),
// complex as 4 real DMMAs on planar operands; each warp owns a 16x16 sub-tile
// (8 independent accumulator chains).
//
//   variant 0  L   forward  (direct solve, after the row gather P B)
//   variant 1  U   backward (direct solve)
//   variant 2  U^H forward  (adjoint solve)
//   variant 3  L^H backward (adjoint solve, then the row scatter P^T)
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "common.cuh"
#include "trsm.cuh"

namespace cg = cooperative_groups;

namespace fb {

namespace {

constexpr int BS = 32;                 // block rows (= PW of the factorization)
constexpr int CW = 32;                 // right-hand-side columns per chunk (64: 1.4x slower on C2, fewer CTAs per SM)
constexpr int WC = CW / 16;            // warps along the columns (16x16 sub-tile each)
constexpr int TT = 32 * 2 * WC;        // threads: 4 warps in a 2x2 grid of 16x16 sub-tiles
constexpr int GT = 128;                // threads of the gmat kernel
constexpr int PA = 36;                 // operator tile pitch (= 4 mod 16: conflict-free fragments, both orientations)
constexpr int XP = CW + 4;             // X tile pitch (= 4 mod 16)
constexpr int TILE = 2 * BS * PA;      // doubles per planar 32x32 operator tile in shared memory
constexpr int XTILE = 2 * BS * XP;     // doubles per planar 32 x CW X tile
constexpr int GM_BLK = 4 * BS * BS;    // per (variant, block): G re/im, D re/im

struct SweepArgs {
  int n, nrhs, nblk, variant;
  const double *lre, *lim;
  long long ld;
  const double* dinv;  // [nblk][L re, L im, U re, U im][32][32]
  const double* gmat;  // [4][nblk][G re, G im, D re, D im][32][32]
  double *xre, *xim;
  long long ldx;
  long long slu, sdinv, sx;  // batch strides (item b: + b * stride)
  int *upd, *fin;             // dataflow counters [count][nblk][C] (zeroed per launch)
};

__device__ __forceinline__ void offset_item(SweepArgs& a, long long b) {
  a.lre += b * a.slu;
  a.lim += b * a.slu;
  a.dinv += b * a.sdinv;
  a.gmat += b * a.sdinv;
  a.xre += b * a.sx;
  a.xim += b * a.sx;
  const long long nc = (long long)a.nblk * ceil_div(a.nrhs, CW);
  a.upd += b * nc;
  a.fin += b * nc;
}

__device__ __forceinline__ int blk_at(const SweepArgs& a, int t) {
  return (a.variant == 0 || a.variant == 2) ? t : a.nblk - 1 - t;
}

// --- cp.async tile loader ---------------------------------------------------------
// Natural copy of the planar block [r0, r0 + 32) x [c0, c0 + NC) of a row-major
// matrix (row stride ld) into a pitch-P tile; rows >= nr / cols >= nc read 0.
template <bool VEC, int NC = BS, int P = PA>
__device__ __forceinline__ void cp_block(const double* re, const double* im, long long ld, int r0, int c0,
                                         int nr, int nc, double* s) {
  if (VEC) {
    for (int e = threadIdx.x; e < BS * NC / 2; e += TT) {
      const int r = e / (NC / 2), c = (e % (NC / 2)) * 2;
      const int gr = r0 + r, gc = c0 + c;
      const int valid = gr < nr ? max(0, min(2, nc - gc)) : 0;
      const long long o = valid ? (long long)gr * ld + gc : 0;
      cp_async16(s + r * P + c, re + o, valid * 8);
      cp_async16(s + BS * P + r * P + c, im + o, valid * 8);
    }
  } else {
    for (int e = threadIdx.x; e < BS * NC; e += TT) {
      const int r = e / NC, c = e % NC;
      const int gr = r0 + r, gc = c0 + c;
      const bool ok = gr < nr && gc < nc;
      const long long o = ok ? (long long)gr * ld + gc : 0;
      cp_async8(s + r * P + c, re + o, ok);
      cp_async8(s + BS * P + r * P + c, im + o, ok);
    }
  }
}

// contiguous 32x32 operator tile (G or D of this variant)
template <bool VEC>
__device__ __forceinline__ void cp_op(const double* src, double* s) {
  cp_block<VEC>(src, src + BS * BS, BS, 0, 0, BS, BS, s);
}

// --- warp sub-tile arithmetic ---------------------------------------------------
// accumulator fragment: rows wr*16 + mt*8 + (lane>>2), cols wc*16 + nt*8 + 2*(lane&3) + e
struct Acc {
  double r[2][2][2], i[2][2][2];
};

__device__ __forceinline__ void acc_zero(Acc& c) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) c.r[mt][nt][e] = c.i[mt][nt][e] = 0.0;
}

// acc += (SR*Re A + i*SI*Im A) (32x32) * B (32 x CW tile of X); A is read as
// A[r][k] = S[r*PA + k] (TR = false) or S[k*PA + r] (TR = true).  The signs
// are compile-time and applied as integer sign-bit flips, so the FP64 pipe
// that issues the DMMAs carries no extra multiplies.  live = false: the
// warp's 16 columns lie past nrhs (warp-uniform skip, no barriers inside).
__device__ __forceinline__ double sgnflip(double v) {
  return __longlong_as_double(__double_as_longlong(v) ^ 0x8000000000000000ll);
}
template <bool TR, int SR, int SI>
__device__ __forceinline__ void tile_mma(Acc& c, const double* A, const double* B, bool live) {
  if (!live) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = w / WC, wc = w % WC;
  const double* Ai = A + BS * PA;
  const double* Bi = B + BS * XP;
#pragma unroll
  for (int k0 = 0; k0 < BS; k0 += 4) {
    const int k = k0 + (lane & 3);
    double ar[2], ai[2], nai[2], br[2], bi[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = wr * 16 + mt * 8 + (lane >> 2);
      const int o = TR ? k * PA + r : r * PA + k;
      const double xr = A[o], xi = Ai[o];
      ar[mt] = SR > 0 ? xr : sgnflip(xr);
      ai[mt] = SI > 0 ? xi : sgnflip(xi);
      nai[mt] = SI > 0 ? sgnflip(xi) : xi;
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int col = wc * 16 + nt * 8 + (lane >> 2);
      br[nt] = B[k * XP + col];
      bi[nt] = Bi[k * XP + col];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        dmma(c.r[mt][nt][0], c.r[mt][nt][1], ar[mt], br[nt]);
        dmma(c.i[mt][nt][0], c.i[mt][nt][1], ar[mt], bi[nt]);
      }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        dmma(c.r[mt][nt][0], c.r[mt][nt][1], nai[mt], bi[nt]);
        dmma(c.i[mt][nt][0], c.i[mt][nt][1], ai[mt], br[nt]);
      }
  }
}

// global X <-> accumulator fragments (L2-only loads: other CTAs wrote X in
// earlier steps)
template <bool VEC>
__device__ __forceinline__ void acc_load(const SweepArgs& a, int b, int c0, Acc& c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = w / WC, wc = w % WC;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int gr = b * BS + wr * 16 + mt * 8 + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int gc = c0 + wc * 16 + nt * 8 + 2 * (lane & 3);
      const long long o = (long long)gr * a.ldx + gc;
      if (VEC && gr < a.n && gc + 1 < a.nrhs) {
        const double2 vr = __ldcg(reinterpret_cast<const double2*>(a.xre + o));
        const double2 vi = __ldcg(reinterpret_cast<const double2*>(a.xim + o));
        c.r[mt][nt][0] = vr.x; c.r[mt][nt][1] = vr.y;
        c.i[mt][nt][0] = vi.x; c.i[mt][nt][1] = vi.y;
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = gr < a.n && gc + e < a.nrhs;
          c.r[mt][nt][e] = ok ? __ldcg(a.xre + o + e) : 0.0;
          c.i[mt][nt][e] = ok ? __ldcg(a.xim + o + e) : 0.0;
        }
      }
    }
  }
}

template <bool VEC>
__device__ __forceinline__ void acc_store(const SweepArgs& a, int b, int c0, const Acc& c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = w / WC, wc = w % WC;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int gr = b * BS + wr * 16 + mt * 8 + (lane >> 2);
    if (gr >= a.n) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int gc = c0 + wc * 16 + nt * 8 + 2 * (lane & 3);
      const long long o = (long long)gr * a.ldx + gc;
      if (VEC && gc + 1 < a.nrhs) {
        __stcg(reinterpret_cast<double2*>(a.xre + o), make_double2(c.r[mt][nt][0], c.r[mt][nt][1]));
        __stcg(reinterpret_cast<double2*>(a.xim + o), make_double2(c.i[mt][nt][0], c.i[mt][nt][1]));
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (gc + e < a.nrhs) {
            __stcg(a.xre + o + e, c.r[mt][nt][e]);
            __stcg(a.xim + o + e, c.i[mt][nt][e]);
          }
      }
    }
  }
}

__device__ __forceinline__ const double* op_ptr(const SweepArgs& a, int b, int which) {
  return a.gmat + ((size_t)a.variant * a.nblk + b) * GM_BLK + which * 2 * BS * BS;  // 0: G, 1: D
}

// X tile rows of block b, chunk columns [c0, c0 + 32).  X is written by other
// CTAs during the sweep, so it is read through L2 only (cp.async.cg, or plain
// .cg loads on the unaligned path).
template <bool VEC>
__device__ __forceinline__ void cp_x(const SweepArgs& a, int b, int c0, double* s) {
  if (VEC) {
    cp_block<true, CW, XP>(a.xre, a.xim, a.ldx, b * BS, c0, a.n, a.nrhs, s);
  } else {
    for (int e = threadIdx.x; e < BS * CW; e += TT) {
      const int r = e / CW, c = e % CW;
      const int gr = b * BS + r, gc = c0 + c;
      const bool ok = gr < a.n && gc < a.nrhs;
      const long long o = (long long)gr * a.ldx + gc;
      s[r * XP + c] = ok ? __ldcg(a.xre + o) : 0.0;
      s[BS * XP + r * XP + c] = ok ? __ldcg(a.xim + o) : 0.0;
    }
  }
}

// streamed operator tile M(i, b) (TR: stored as the natural block LU(b, i))
template <bool VEC>
__device__ __forceinline__ void cp_m(const SweepArgs& a, int bi, int bb, double* s) {
  if (a.variant < 2)
    cp_block<VEC>(a.lre, a.lim, a.ld, bi * BS, bb * BS, a.n, a.n, s);
  else
    cp_block<VEC>(a.lre, a.lim, a.ld, bb * BS, bi * BS, a.n, a.n, s);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  while (ld_acquire(p) < v) __nanosleep(20);
}
// after a __syncthreads that follows the tile stores: publish (thread 0)
__device__ __forceinline__ void publish(int* p, int v) {
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(p, v);
  }
}

// Dataflow schedule (no grid barriers).  Per (row block i, chunk c):
//   upd[i][c] = number of streamed rank-32 updates applied so far,
//   fin[i][c] = 1 once X_i[:, c] is final.
// Step t: the look-ahead for b(t+1) needs fin[b(t)] and upd[b(t+1)] == t;
// the streamed update of row block i needs fin[b(t)] and upd[i] == t.  Every
// wait points at an earlier step and CTAs walk the steps in order, so with
// all CTAs co-resident (cooperative launch) the schedule cannot deadlock.
// Sub-CTA 0 of a chunk group owns the critical chain (look-ahead + the next
// row block); the others stream the remaining rows and may run ahead.
template <bool TR, bool VEC>
__device__ void sweep_body(SweepArgs& a, double* s) {
  const int G = gridDim.x, g = blockIdx.x;
  const int C = ceil_div(a.nrhs, CW);
  // chunk group of this CTA: one chunk if G >= C, else chunks g, g + G, ...
  const int S = G >= C ? G / C + (g % C < G % C ? 1 : 0) : 1;
  const int sub = G >= C ? g / C : 0;
  double* Xt = s;                      // X_{b(t)} chunk (B operand of every product this step)
  double* Xn = s + XTILE;              // X_{b(t+1)} chunk (look-ahead)
  double* T0 = s + 2 * XTILE;          // operator stage 0
  double* T1 = s + 2 * XTILE + TILE;   // operator stage 1
  const int wcol = ((threadIdx.x >> 5) % WC) * 16;  // this warp's first column inside a chunk
  auto upd = [&](int blk, int c) { return a.upd + (size_t)blk * C + c; };
  auto fin = [&](int blk, int c) { return a.fin + (size_t)blk * C + c; };
  const int c_first = G >= C ? g % C : g, c_step = G >= C ? C : G;

  // prologue: the first block of the sweep is final after D
  if (sub == 0) {
    const int b0 = blk_at(a, 0);
    for (int c = c_first; c < C; c += c_step) {
      cp_op<VEC>(op_ptr(a, b0, 1), T0);
      cp_x<VEC>(a, b0, c * CW, Xt);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      Acc acc;
      acc_zero(acc);
      tile_mma<false, 1, 1>(acc, T0, Xt, c * CW + wcol < a.nrhs);
      acc_store<VEC>(a, b0, c * CW, acc);
      __syncthreads();
      publish(fin(b0, c), 1);
    }
  }

  for (int t = 0; t < a.nblk; ++t) {
    const int bt = blk_at(a, t);
    const bool ahead = t + 1 < a.nblk;
    const int R = max(0, a.nblk - t - 2);  // pending row blocks b(t+2) ...
    // units: [0, 2) = look-ahead (weight of two products), then one per
    // pending row block; sub-CTA s takes units [s*U/S, (s+1)*U/S), so sub 0
    // holds the look-ahead and the nearest rows (the critical chain).
    // (Weighting the look-ahead so that sub 0 holds nothing else measured
    // 10-20 % slower on C2/C3: throughput, not the chain, bounds the sweep.)
    const int U = R + (ahead ? 2 : 0), u_off = ahead ? 2 : 0;
    const int ub = (int)((long long)sub * U / S), ue = (int)((long long)(sub + 1) * U / S);
    const int qb = max(ub - u_off, 0), qe = max(ue - u_off, 0);
    const bool do_ahead = ahead && ub == 0 && ue > 0;
    if (!do_ahead && qb >= qe) continue;
    for (int c = c_first; c < C; c += c_step) {
      const int c0 = c * CW;
      const bool live = c0 + wcol < a.nrhs;
      if (threadIdx.x == 0) wait_ge(fin(bt, c), 1);
      if (do_ahead && threadIdx.x == 32) wait_ge(upd(blk_at(a, t + 1), c), t);
      __syncthreads();
      cp_x<VEC>(a, bt, c0, Xt);
      if (do_ahead) {
        const int bn = blk_at(a, t + 1);
        cp_x<VEC>(a, bn, c0, Xn);
        cp_op<VEC>(op_ptr(a, bn, 1), T0);
        cp_op<VEC>(op_ptr(a, bn, 0), T1);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        Acc acc;
        acc_zero(acc);
        tile_mma<false, 1, 1>(acc, T0, Xn, live);
        tile_mma<false, -1, -1>(acc, T1, Xt, live);
        acc_store<VEC>(a, bn, c0, acc);
        __syncthreads();
        publish(fin(bn, c), 1);
      }
      if (qb < qe) {
        // the rows' previous-step updates
        for (int q = qb + threadIdx.x; q < qe; q += TT) wait_ge(upd(blk_at(a, t + 2 + q), c), t);
        __syncthreads();
        Acc cur, nxt;
        cp_m<VEC>(a, blk_at(a, t + 2 + qb), bt, T0);
        cp_async_commit();
        acc_load<VEC>(a, blk_at(a, t + 2 + qb), c0, nxt);
        for (int q = qb; q < qe; ++q) {
          const int rb = blk_at(a, t + 2 + q);
          double* Tq = ((q - qb) & 1) ? T1 : T0;
          cur = nxt;
          if (q + 1 < qe) {
            const int rn = blk_at(a, t + 3 + q);
            cp_m<VEC>(a, rn, bt, ((q - qb) & 1) ? T0 : T1);
            cp_async_commit();
            acc_load<VEC>(a, rn, c0, nxt);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          __syncthreads();
          tile_mma<TR, -1, (TR ? 1 : -1)>(cur, Tq, Xt, live);
          acc_store<VEC>(a, rb, c0, cur);
          __syncthreads();
        }
        // one fence for the CTA's rows of this step, then the counters
        if (threadIdx.x == 0) {
          __threadfence();
          for (int q = qb; q < qe; ++q) st_relaxed(upd(blk_at(a, t + 2 + q), c), t + 1);
        }
      }
      cp_async_wait<0>();
      __syncthreads();  // Xt is restaged by the next chunk / step
    }
  }
}

template <bool TR, bool VEC>
__global__ void __launch_bounds__(TT) sweep_kernel(SweepArgs a0) {
  extern __shared__ __align__(16) double s[];
  SweepArgs a = a0;
  offset_item(a, blockIdx.y);
  sweep_body<TR, VEC>(a, s);
}

// Per (block, variant): D_v (the variant's diagonal inverse, conj-transposed for
// the adjoint sweeps) and G_v = D_v * M(b, prev(b)).
__global__ void __launch_bounds__(GT) gmat_kernel(SweepArgs a0) {
  __shared__ double Dr[BS * 33], Di[BS * 33], Mr[BS * 33], Mi[BS * 33];
  SweepArgs a = a0;
  offset_item(a, blockIdx.z);
  const int b = blockIdx.x, variant = blockIdx.y;
  const bool upper = variant == 1 || variant == 2;
  const bool trans = variant >= 2;
  const double* dr = a.dinv + (size_t)b * 4 * BS * BS + (upper ? 2 : 0) * BS * BS;
  const double* di = dr + BS * BS;
  double* out = const_cast<double*>(a.gmat) + ((size_t)variant * a.nblk + b) * GM_BLK;
  for (int e = threadIdx.x; e < BS * BS; e += GT) {
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
    for (int e = threadIdx.x; e < BS * BS; e += GT) out[e] = out[BS * BS + e] = 0.0;
    return;
  }
  const int i0 = b * BS, p0 = prev * BS;
  for (int e = threadIdx.x; e < BS * BS; e += GT) {
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
  for (int e = threadIdx.x; e < BS * BS; e += GT) {
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

size_t sweep_smem() { return sizeof(double) * (2 * XTILE + 2 * TILE); }

}  // namespace

size_t gmat_doubles(int n) { return (size_t)4 * ceil_div(n, BS) * GM_BLK; }

cudaError_t gmat_launch(int n, int count, const double* lre, const double* lim, long long ld, long long slu,
                        const double* dinv, long long sdinv, double* gmat, cudaStream_t st) {
  SweepArgs a{};
  a.n = n; a.nblk = ceil_div(n, BS); a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.slu = slu; a.sdinv = sdinv; a.sx = 0;
  gmat_kernel<<<dim3(a.nblk, 4, count), GT, 0, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t sweep_launch_one(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                                    long long ld, long long slu, const double* dinv, const double* gmat,
                                    long long sdinv, double* xre, double* xim, long long ldx, long long sx,
                                    cudaStream_t st);

// The right-hand sides of all items are read and rewritten by every step
// (right-looking accumulators), so the batch is swept in groups whose
// accumulators fit in L2 (FB_SWEEP_L2MB, default 64 MB): past that the
// accumulator traffic spills to HBM (C3: 321 MB of X for 16 shifts).
cudaError_t sweep_launch(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                         long long ld, long long slu, const double* dinv, const double* gmat, long long sdinv,
                         double* xre, double* xim, long long ldx, long long sx, cudaStream_t st) {
  if (n <= 0 || nrhs <= 0 || count <= 0) return cudaSuccess;
  static const double budget = 1048576.0 * (getenv("FB_SWEEP_L2MB") ? atof(getenv("FB_SWEEP_L2MB")) : 64.0);
  const double item = 16.0 * (double)n * (double)nrhs;
  int group = count;
  if (count * item > 1.5 * budget) {  // C2's 84 MB stays one launch; C3's 321 MB goes in 3-shift groups
    const int per = std::max(1, (int)(budget / item));
    group = ceil_div(count, ceil_div(count, per));  // balanced
  }
  for (int b0 = 0; b0 < count; b0 += group) {
    const int cnt = std::min(group, count - b0);
    cudaError_t e = sweep_launch_one(variant, n, nrhs, cnt, lre + b0 * slu, lim + b0 * slu, ld, slu,
                                     dinv + b0 * sdinv, gmat + b0 * sdinv, sdinv, xre + b0 * sx, xim + b0 * sx,
                                     ldx, sx, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static cudaError_t sweep_launch_one(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                                    long long ld, long long slu, const double* dinv, const double* gmat,
                                    long long sdinv, double* xre, double* xim, long long ldx, long long sx,
                                    cudaStream_t st) {
  SweepArgs a{};
  a.n = n; a.nrhs = nrhs; a.nblk = ceil_div(n, BS); a.variant = variant;
  a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.xre = xre; a.xim = xim; a.ldx = ldx;
  a.slu = slu; a.sdinv = sdinv; a.sx = sx;
  // 16-byte paths need every row start 16-byte aligned
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool vec = ld % 2 == 0 && ldx % 2 == 0 && slu % 2 == 0 && sx % 2 == 0 && sdinv % 2 == 0 &&
                   al(lre) && al(lim) && al(xre) && al(xim) && al(gmat);
  const bool tr = variant >= 2;
  void* fn = tr ? (vec ? (void*)sweep_kernel<true, true> : (void*)sweep_kernel<true, false>)
                : (vec ? (void*)sweep_kernel<false, true> : (void*)sweep_kernel<false, false>);
  const int ki = (tr ? 2 : 0) + (vec ? 1 : 0);
  static int blocks[4] = {0, 0, 0, 0};
  const size_t smem = sweep_smem();
  if (blocks[ki] == 0) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, TT, smem);
    blocks[ki] = std::max(1, nb);
  }
  const int C = ceil_div(nrhs, CW);
  const int cap = (blocks[ki] * kSMs) / count;
  if (cap < 1) return cudaErrorInvalidValue;
  // enough CTAs per chunk group to spread the pending rows, whole groups when possible
  const int want = C * std::max(1, ceil_div(a.nblk, 2));
  int G = std::min(cap, want);
  if (G > C) G -= G % C;
  G = std::max(G, 1);
  // dataflow counters (upd, fin), zeroed on the stream before the sweep
  const size_t cnt = (size_t)2 * count * a.nblk * C;
  int* ctr = nullptr;
  {
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, std::pair<int*, size_t>> bufs;
    std::lock_guard<std::mutex> lk(mu);
    auto& b = bufs[st];
    if (b.second < cnt) {
      if (b.first) cudaFree(b.first);
      b.first = nullptr;
      b.second = 0;
      cudaError_t e = cudaMalloc(&b.first, cnt * sizeof(int));
      if (e != cudaSuccess) return e;
      b.second = cnt;
    }
    ctr = b.first;
  }
  cudaError_t e = cudaMemsetAsync(ctr, 0, cnt * sizeof(int), st);
  if (e != cudaSuccess) return e;
  a.upd = ctr;
  a.fin = ctr + cnt / 2;
  void* args[] = {&a};
  count_launch();
  return cudaLaunchCooperativeKernel(fn, dim3(G, count), dim3(TT), args, smem, st);
}

}  // namespace fb
