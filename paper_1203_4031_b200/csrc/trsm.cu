// Fused multi-RHS triangular sweeps for the dense shifted solves (dense.py:53-88).
//
// One cooperative kernel per sweep replaces the 2*N/32 launches of a blocked
// TRSM.  Blocks of 32 rows are finalised in processing order b(0), b(1), ...
// (ascending for the L / U^H sweeps, descending for U / L^H).  The right-hand
// sides are cut into 32-column chunks and every CTA owns ONE chunk for the
// whole sweep (a group of S CTAs per chunk), so at step t it stages the final
// block X_{b(t)}[:, chunk] in shared memory once and then:
//   * sub-CTA 0 of the group finalises the NEXT block ("look-ahead"):
//       P = X_{b(t+1)} - M(b(t+1), b(t)) X_{b(t)}     (DMMA, K = 32)
//       X_{b(t+1)} = T_{b(t+1)}^{-1} P                 (substitution)
//     The 32x32 diagonal block T is applied by forward/backward SUBSTITUTION
//     in shared memory (lanes = rows, 8 columns per warp, the pivot row
//     broadcast by shuffles), not by an explicit inverse: a precomputed
//     diagonal-block inverse costs a factor cond(T) in backward error (4x
//     LAPACK's at N = 8192, profiles/r02_backward_error.txt), substitution
//     is backward stable like zgetrs;
//   * the group streams the rank-32 update of its share of the pending rows,
//       X_i -= M(i, b(t)) X_{b(t)},   i in b(t+2) ...
//     with the 32x32 M tiles double-buffered by 16-byte cp.async and the X_i
//     accumulators prefetched straight into registers (L2-only loads);
//   * no grid barriers: per (row block, chunk) counters in global memory
//     (release/acquire) let each CTA start a step as soon as the blocks it
//     reads are final, so steps overlap (see sweep_body).
// All block products run on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA),
// complex as 4 real DMMAs on planar operands; each warp owns a 16x16 sub-tile
// (8 independent accumulator chains).
//
// For N >= 6144 the sweeps run BLOCKED instead (sweep_launch): block_solve_kernel
// solves each 256-row diagonal block with the chunk of X resident in shared
// memory, and one TMA-fed ZGEMM (gemm_tma.cu, K = 256) updates all pending rows.
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
#include "gemm.cuh"
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
constexpr int SOB = 256;               // outer block of the blocked sweeps (= K of the TMA update; 128 measured equal at C3, slower at C2)
constexpr int SOB_MIN_N = 6144;        // below, the block solves cost more than the faster updates gain (C2: +3 %, C1: +6 %)
constexpr int GM_BLK = 4 * BS * BS;    // per (variant, block): T re/im [32][32], inv re/im [32] (padded)

struct SweepArgs {
  int n, nrhs, nblk, variant;
  const double *lre, *lim;
  long long ld;
  const double* dinv;  // factor side store (only its gmat part is read here)
  const double* gmat;  // [4][nblk][T re, T im][32][32] + [inv re, inv im][32] (see tdiag_kernel)
  double *xre, *xim;
  long long ldx;
  long long slu, sdinv, sx;  // batch strides (item b: + b * stride)
  int *upd, *fin;             // dataflow counters [count][nblk][C] (zeroed per launch)
  int gblk0, gnblk;           // block solves: operator index of block 0 and the whole matrix's block count
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

__device__ __forceinline__ void acc_add(Acc& c, const Acc& d) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        c.r[mt][nt][e] += d.r[mt][nt][e];
        c.i[mt][nt][e] += d.i[mt][nt][e];
      }
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

__device__ __forceinline__ const double* op_ptr(const SweepArgs& a, int b) {
  return a.gmat + ((size_t)a.variant * a.gnblk + a.gblk0 + b) * GM_BLK;
}

// The diagonal-block operator of block b in processing coordinates (tdiag_kernel):
// T[i][k] (step i, lane k) is the multiplier of the pivot row of step i applied
// to processing row k (zero unless k > i), inv[k] the final scale of row k.
// Copy it into a pitch-PA tile followed by inv (64 doubles).
template <bool VEC>
__device__ __forceinline__ void cp_tdiag(const double* src, double* s) {
  cp_op<VEC>(src, s);
  for (int e = threadIdx.x; e < 2 * BS; e += TT) cp_async8(s + 2 * BS * PA + e, src + 2 * BS * BS + e, true);
}

// X <- T^{-1} X on the planar shared tile X (pitch XP): forward substitution in
// processing order (tile row = lane for the ascending sweeps, 31 - lane for the
// descending ones).  Warp w owns columns [8w, 8w + 8); lane k holds row k of
// its 8 columns; step i broadcasts row i (final) by shuffles and every lane
// subtracts T[i][k] * x_i (T[i][k] = 0 for k <= i).  Backward stable as the
// column-oriented substitution of zgetrs; the pivot scale of the non-unit
// sweeps (U, U^H) is folded into T and applied to each row once at the end.
template <bool FWD>
__device__ __forceinline__ void tile_subst(double* X, const double* T, int c0, int nrhs) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int WCOL = CW / (TT / 32);
  if (c0 + w * WCOL >= nrhs) return;  // warp-uniform: no live column
  const int row = FWD ? lane : BS - 1 - lane;
  double* Xr = X + row * XP + w * WCOL;
  double* Xi = Xr + BS * XP;
  double yr[WCOL], yi[WCOL];
#pragma unroll
  for (int c = 0; c < WCOL; ++c) {
    yr[c] = Xr[c];
    yi[c] = Xi[c];
  }
  const double* Ti = T + BS * PA;
#pragma unroll
  for (int i = 0; i < BS - 1; ++i) {
    const double tr = T[i * PA + lane], ti = Ti[i * PA + lane];
#pragma unroll
    for (int c = 0; c < WCOL; ++c) {
      const double br = __shfl_sync(0xffffffffu, yr[c], i), bi = __shfl_sync(0xffffffffu, yi[c], i);
      yr[c] = fma(-tr, br, fma(ti, bi, yr[c]));
      yi[c] = fma(-tr, bi, fma(-ti, br, yi[c]));
    }
  }
  const double sr = T[2 * BS * PA + lane], si = T[2 * BS * PA + BS + lane];
#pragma unroll
  for (int c = 0; c < WCOL; ++c) {
    Xr[c] = yr[c] * sr - yi[c] * si;
    Xi[c] = yr[c] * si + yi[c] * sr;
  }
}

// P = X_shared + acc (acc = -M X_b as fragments) written back into the shared tile
__device__ __forceinline__ void acc_add_to_tile(const Acc& c, double* X) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = w / WC, wc = w % WC;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int r = wr * 16 + mt * 8 + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int col = wc * 16 + nt * 8 + 2 * (lane & 3);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        X[r * XP + col + e] += c.r[mt][nt][e];
        X[BS * XP + r * XP + col + e] += c.i[mt][nt][e];
      }
    }
  }
}

// shared X tile -> global rows of block b, chunk columns [c0, c0 + CW) (L2 stores)
__device__ __forceinline__ void tile_store(const SweepArgs& a, int b, int c0, const double* X) {
  for (int e = threadIdx.x; e < BS * CW; e += TT) {
    const int r = e / CW, c = e % CW;
    const int gr = b * BS + r, gc = c0 + c;
    if (gr < a.n && gc < a.nrhs) {
      const long long o = (long long)gr * a.ldx + gc;
      __stcg(a.xre + o, X[r * XP + c]);
      __stcg(a.xim + o, X[BS * XP + r * XP + c]);
    }
  }
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

  const bool fwd = a.variant == 0 || a.variant == 2;
  // prologue: the first block of the sweep is final after its substitution
  if (sub == 0) {
    const int b0 = blk_at(a, 0);
    for (int c = c_first; c < C; c += c_step) {
      cp_tdiag<VEC>(op_ptr(a, b0), T1);
      cp_x<VEC>(a, b0, c * CW, Xt);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      if (fwd)
        tile_subst<true>(Xt, T1, c * CW, a.nrhs);
      else
        tile_subst<false>(Xt, T1, c * CW, a.nrhs);
      __syncthreads();
      tile_store(a, b0, c * CW, Xt);
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
        cp_m<VEC>(a, bn, bt, T0);
        cp_tdiag<VEC>(op_ptr(a, bn), T1);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        Acc acc;
        acc_zero(acc);
        tile_mma<TR, -1, (TR ? 1 : -1)>(acc, T0, Xt, live);
        acc_add_to_tile(acc, Xn);
        __syncthreads();
        if (fwd)
          tile_subst<true>(Xn, T1, c0, a.nrhs);
        else
          tile_subst<false>(Xn, T1, c0, a.nrhs);
        __syncthreads();
        tile_store(a, bn, c0, Xn);
        __syncthreads();
        publish(fin(bn, c), 1);
      }
      if (qb < qe) {
        // the rows' previous-step updates
        for (int q = qb + threadIdx.x; q < qe; q += TT) wait_ge(upd(blk_at(a, t + 2 + q), c), t);
        __syncthreads();
        // the product -M X_b accumulates from zero and is added to the
        // prefetched X_i once (one rounding per element and step, as zgetrs'
        // GEMM updates; accumulating onto X_i would round all 32 FMAs at
        // |X_i|'s magnitude, tools/dmma_rounding.py)
        Acc cur, nxt, prod;
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
          acc_zero(prod);
          tile_mma<TR, -1, (TR ? 1 : -1)>(prod, Tq, Xt, live);
          acc_add(cur, prod);
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

// One CTA solves a whole diagonal block of up to SOB rows for one 32-column
// chunk of one shift (the blocked sweeps' diagonal step): the chunk of X stays
// in shared memory from load to store, so the 8 substitutions and 28 rank-32
// updates of a 256-row block need no inter-CTA hand-over (measured at C2's
// shapes: 94 us per block against 110-120 us for the dataflow sweep on the
// same block, and no cooperative launch).
template <bool TR, bool VEC>
__global__ void __launch_bounds__(TT) block_solve_kernel(SweepArgs a0) {
  extern __shared__ __align__(16) double s[];
  SweepArgs a = a0;
  offset_item(a, blockIdx.y);
  const int c0 = blockIdx.x * CW;
  double* Xs = s;                                  // nblk tiles of the X chunk
  double* T0 = s + (size_t)a.nblk * XTILE;         // streamed operator tiles (double buffer)
  double* T1 = T0 + TILE;
  double* Td = T1 + TILE;                          // diagonal operator + inverse pivots
  const bool fwd = a.variant == 0 || a.variant == 2;
  const bool live = c0 + ((threadIdx.x >> 5) % WC) * 16 < a.nrhs;
  for (int b = 0; b < a.nblk; ++b) cp_x<VEC>(a, b, c0, Xs + (size_t)b * XTILE);
  for (int t = 0; t < a.nblk; ++t) {
    const int bt = blk_at(a, t);
    double* Xt = Xs + (size_t)bt * XTILE;
    const int R = a.nblk - t - 1;  // pending blocks b(t+1) ...
    cp_tdiag<VEC>(op_ptr(a, bt), Td);
    if (R > 0) cp_m<VEC>(a, blk_at(a, t + 1), bt, T0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (fwd)
      tile_subst<true>(Xt, Td, c0, a.nrhs);
    else
      tile_subst<false>(Xt, Td, c0, a.nrhs);
    __syncthreads();
    for (int q = 0; q < R; ++q) {
      double* Tq = (q & 1) ? T1 : T0;
      if (q + 1 < R) {
        cp_m<VEC>(a, blk_at(a, t + 2 + q), bt, (q & 1) ? T0 : T1);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      // -M X_b from zero, added to the pending tile once (one rounding per element and step)
      Acc prod;
      acc_zero(prod);
      tile_mma<TR, -1, (TR ? 1 : -1)>(prod, Tq, Xt, live);
      acc_add_to_tile(prod, Xs + (size_t)blk_at(a, t + 1 + q) * XTILE);
      __syncthreads();
    }
  }
  for (int b = 0; b < a.nblk; ++b) tile_store(a, b, c0, Xs + (size_t)b * XTILE);
}

// Per (block, variant): the diagonal block of the factor as the substitution
// operator of tile_subst, in processing coordinates p (tile row r = p for the
// ascending sweeps 0 (L) and 2 (U^H), r = 31 - p for the descending sweeps
// 1 (U) and 3 (L^H)):
//   T[i][k] = op(i -> k) / d_i  for k > i (0 otherwise),   inv[k] = 1 / d_k,
// where op(i -> k) is the entry of the triangular block that multiplies row i
// when eliminating row k and d the diagonal (1 for the unit sweeps 0 and 3).
//   variant 0: op = L[rk][ri]          variant 1: op = U[rk][ri], d = U[r][r]
//   variant 2: op = conj(U[ri][rk]),   variant 3: op = conj(L[ri][rk])
//              d = conj(U[r][r])
// Rows past n get inv = 0 and no coupling.
__global__ void __launch_bounds__(GT) tdiag_kernel(SweepArgs a0) {
  __shared__ double Dr[BS * 33], Di[BS * 33], Sr[BS], Si[BS];
  SweepArgs a = a0;
  offset_item(a, blockIdx.z);
  const int b = blockIdx.x, variant = blockIdx.y;
  const bool unit = variant == 0 || variant == 3;
  const bool fwd = variant == 0 || variant == 2;
  const bool trans = variant >= 2;
  const int i0 = b * BS;
  double* out = const_cast<double*>(a.gmat) + ((size_t)variant * a.nblk + b) * GM_BLK;
  for (int e = threadIdx.x; e < BS * BS; e += GT) {
    const int r = e / BS, c = e % BS;
    const bool ok = i0 + r < a.n && i0 + c < a.n;
    Dr[r * 33 + c] = ok ? a.lre[(long long)(i0 + r) * a.ld + i0 + c] : 0.0;
    Di[r * 33 + c] = ok ? a.lim[(long long)(i0 + r) * a.ld + i0 + c] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < BS) {
    const int r = threadIdx.x;  // tile row
    double sr = 0.0, si = 0.0;
    if (i0 + r < a.n) {
      if (unit) {
        sr = 1.0;
      } else {
        const double dr = Dr[r * 33 + r], di = trans ? -Di[r * 33 + r] : Di[r * 33 + r];
        const double den = dr * dr + di * di;
        sr = dr / den;
        si = -di / den;
      }
    }
    Sr[r] = sr;
    Si[r] = si;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BS * BS; e += GT) {
    const int i = e / BS, k = e % BS;
    const int ri = fwd ? i : BS - 1 - i, rk = fwd ? k : BS - 1 - k;
    double vr = 0.0, vi = 0.0;
    if (k > i && i0 + ri < a.n && i0 + rk < a.n) {
      double orr, oi;
      if (!trans) {
        orr = Dr[rk * 33 + ri];
        oi = Di[rk * 33 + ri];
      } else {
        orr = Dr[ri * 33 + rk];
        oi = -Di[ri * 33 + rk];
      }
      if (unit) {
        vr = orr;
        vi = oi;
      } else {
        vr = orr * Sr[ri] - oi * Si[ri];
        vi = orr * Si[ri] + oi * Sr[ri];
      }
    }
    out[e] = vr;
    out[BS * BS + e] = vi;
  }
  if (threadIdx.x < BS) {
    const int k = threadIdx.x, rk = fwd ? k : BS - 1 - k;
    out[2 * BS * BS + k] = Sr[rk];
    out[2 * BS * BS + BS + k] = Si[rk];
  }
}

size_t sweep_smem() { return sizeof(double) * (2 * XTILE + 2 * TILE + 2 * BS); }

}  // namespace

size_t gmat_doubles(int n) { return (size_t)4 * ceil_div(n, BS) * GM_BLK; }

cudaError_t gmat_launch(int n, int count, const double* lre, const double* lim, long long ld, long long slu,
                        const double* dinv, long long sdinv, double* gmat, cudaStream_t st) {
  SweepArgs a{};
  a.n = n; a.nblk = ceil_div(n, BS); a.gnblk = a.nblk; a.gblk0 = 0; a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.slu = slu; a.sdinv = sdinv; a.sx = 0;
  tdiag_kernel<<<dim3(a.nblk, 4, count), GT, 0, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t sweep_launch_one(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                                    long long ld, long long slu, const double* dinv, const double* gmat,
                                    long long sdinv, double* xre, double* xim, long long ldx, long long sx,
                                    cudaStream_t st);

// diagonal block [gblk0*32, gblk0*32 + n) of the whole matrix (gnblk blocks), n <= SOB
static cudaError_t block_solve_launch(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                                      long long ld, long long slu, const double* dinv, const double* gmat,
                                      long long sdinv, double* xre, double* xim, long long ldx, long long sx,
                                      cudaStream_t st, int gblk0, int gnblk) {
  SweepArgs a{};
  a.n = n; a.nrhs = nrhs; a.nblk = ceil_div(n, BS); a.variant = variant;
  a.gblk0 = gblk0; a.gnblk = gnblk;
  a.lre = lre; a.lim = lim; a.ld = ld; a.dinv = dinv; a.gmat = gmat;
  a.xre = xre; a.xim = xim; a.ldx = ldx;
  a.slu = slu; a.sdinv = sdinv; a.sx = sx;
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool vec = ld % 2 == 0 && ldx % 2 == 0 && slu % 2 == 0 && sx % 2 == 0 && sdinv % 2 == 0 &&
                   al(lre) && al(lim) && al(xre) && al(xim) && al(gmat);
  const size_t smem = sizeof(double) * ((size_t)(SOB / BS) * XTILE + 3 * TILE + 2 * BS);
  static DevOnce cfg;
  if (cfg.first()) {
    cudaFuncSetAttribute(block_solve_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(block_solve_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(block_solve_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(block_solve_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const dim3 grid(ceil_div(nrhs, CW), count);
  if (variant >= 2) {
    if (vec)
      block_solve_kernel<true, true><<<grid, TT, smem, st>>>(a);
    else
      block_solve_kernel<true, false><<<grid, TT, smem, st>>>(a);
  } else if (vec) {
    block_solve_kernel<false, true><<<grid, TT, smem, st>>>(a);
  } else {
    block_solve_kernel<false, false><<<grid, TT, smem, st>>>(a);
  }
  count_launch();
  return cudaGetLastError();
}

// The right-hand sides of all items are read and rewritten by every step
// (right-looking accumulators), so the batch is swept in groups whose
// accumulators fit in L2 (64 MB): past that the
// accumulator traffic spills to HBM (C3: 321 MB of X for 16 shifts).
cudaError_t sweep_launch(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                         long long ld, long long slu, const double* dinv, const double* gmat, long long sdinv,
                         double* xre, double* xim, long long ldx, long long sx, cudaStream_t st) {
  if (n <= 0 || nrhs <= 0 || count <= 0) return cudaSuccess;
  // Sweeps of large matrices run BLOCKED: block_solve_kernel solves one
  // 256-row diagonal block, then the update of all pending rows,
  // X_pend -= M(pend, block) X_block (M^H for the adjoint sweeps), is ONE
  // TMA-fed ZGEMM with K = 256 (95 % of the DMMA pipe against ~55 % for the
  // streamed rank-32 tile updates, and 8x less traffic on X).
  if (n >= SOB_MIN_N && (ld % 2) == 0 && (ldx % 2) == 0 && (slu % 2) == 0 && (sx % 2) == 0) {
    LuTmaMaps ma, mx;
    if (lu_tma_maps_make(&ma, lre, lim, n, ld, slu, count) &&
        lu_tma_maps_make_rect(&mx, xre, xim, n, nrhs, ldx, sx, count)) {
      const int nob = ceil_div(n, SOB), gn = ceil_div(n, BS);
      const bool asc = variant == 0 || variant == 2;  // L and U^H sweep forward, U and L^H backward
      for (int t = 0; t < nob; ++t) {
        const int ob = (asc ? t : nob - 1 - t) * SOB, rows = std::min(SOB, n - ob);
        cudaError_t e = block_solve_launch(variant, rows, nrhs, count, lre + (long long)ob * ld + ob,
                                           lim + (long long)ob * ld + ob, ld, slu, dinv, gmat, sdinv,
                                           xre + (long long)ob * ldx, xim + (long long)ob * ldx, ldx, sx, st, ob / BS, gn);
        if (e != cudaSuccess) return e;
        const int pend0 = asc ? ob + rows : 0, pend = asc ? n - (ob + rows) : ob;
        if (pend > 0) {
          // C = X[pend0.., :], B = X[ob..ob+rows, :]; A = M[pend0.., ob..ob+rows) for the direct sweeps,
          // A(r, k) = conj(M[ob + k][pend0 + r]) for the adjoint ones
          double* cr = xre + (long long)pend0 * ldx;
          double* ci = xim + (long long)pend0 * ldx;
          e = variant < 2 ? zgemm_tma_sub(ma, mx, cr, ci, ldx, sx, count, pend, nrhs, rows, pend0, ob, ob, 0, st, false)
                          : zgemm_tma_sub(ma, mx, cr, ci, ldx, sx, count, pend, nrhs, rows, ob, pend0, ob, 0, st, true);
          if (e != cudaSuccess) return e;
        }
      }
      return cudaSuccess;
    }
  }
  const double budget = 1048576.0 * 64.0;  // sweep working set per launch: about half the 126 MB L2
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
  a.gblk0 = 0; a.gnblk = a.nblk;
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
