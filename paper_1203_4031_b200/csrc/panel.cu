// Sub-panel factorization of the blocked shifted LU (restates dense.py:40-49
// for PW = 32 columns at a time).
//
// The panel rows [c0, n) x [c0, c0+pw) live in shared memory, split across the
// CTAs of a thread-block cluster (<= 16 CTAs, records exchanged through DSMEM,
// one barrier.cluster per column) or, for panels taller than the cluster's
// shared memory, across a cooperative grid (records through L2, one grid
// barrier per column).  Per column j:
//   1. every thread scans its rows for max |a(r, j)| (np.abs = hypot; first
//      index wins ties, as np.argmax, dense.py:41); warp shuffles + one
//      barrier give the CTA candidate, whose full panel row is published
//      together with the current row rj (owner only);
//   2. barrier.cluster / grid barrier;
//   3. warp 0 reduces the <= 16 (or G) candidates and fetches the pivot row and
//      the old row rj (DSMEM / L2);
//   4. each row thread scales its multiplier l = a(r, j) / pivot (rows p and rj
//      take their swapped contents first);
//   5. all threads apply the rank-1 update over the flattened (row, column)
//      space of the remaining panel columns.
// At the end CTA 0 emits the inverses of the 32x32 unit-lower and upper
// diagonal blocks and the (dst, src) list of the panel's row interchanges.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "panel.cuh"

namespace cg = cooperative_groups;

namespace fb {

namespace {

constexpr int PW = PANEL_W;
constexpr int PT = 256;          // threads per panel CTA (8 warps)
constexpr int NW = PT / 32;
constexpr int SP = PW + 1;       // row pitch of the panel in smem (conflict-free per-row access)
constexpr int REC = 2 + 2 * PW;  // exchange record: |pivot|, row, row data (re, im)
constexpr int SB = 8;            // sub-block width: per-column updates stay inside it
constexpr int MAXG = 16;         // max cluster size (mailbox slots)

struct Best {
  double v;
  int r;
};
__device__ __forceinline__ Best better(Best a, Best b) {
  if (b.v > a.v || (b.v == a.v && b.r < a.r)) return b;
  return a;
}
// Warp argmax of (v, row) with exact double comparison and smallest-row ties,
// as three 32-bit redux.sync steps (v >= 0 for candidates, v = -1 for none).
__device__ __forceinline__ Best warp_best(Best b) {
  const unsigned long long k = b.v >= 0.0 ? (unsigned long long)__double_as_longlong(b.v) : 0ull;
  const unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = hi == mhi && lo == mlo;
  const unsigned mr = __reduce_min_sync(0xffffffffu, top ? (unsigned)b.r : 0x7fffffffu);
  Best o;
  o.r = (int)mr;
  o.v = (mr == 0x7fffffffu) ? -1.0 : __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
  return o;
}

// Column `c` of the inverse of the unit-lower (LOWER) or upper diagonal block
// held in rows 0..pw-1 of the CTA's panel.  Rows are produced in blocks of 8
// (from the top for LOWER, from the bottom for the upper block): the terms of
// the rows already finished are summed for all 8 rows of a block at once
// (8 independent accumulators), so only the short in-block recurrence is a
// dependent chain.  This sits on the panel's critical path (the next GEMM
// needs the inverse): the row-at-a-time form cost ~35 us per panel.
template <bool LOWER>
__device__ void tri_inverse(const PanelArgs& a, const double* sre, const double* sim, int c) {
  constexpr int RB = 8;
  double xr[PW], xi[PW];
#pragma unroll
  for (int blk = 0; blk < PW / RB; ++blk) {
    double ar[RB], ai[RB];
    // rows of this block: i(rr) = LOWER ? blk*RB + rr : PW-1 - (blk*RB + rr)
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = LOWER ? blk * RB + rr : PW - 1 - (blk * RB + rr);
      ar[rr] = (i == c) ? 1.0 : 0.0;
      ai[rr] = 0.0;
    }
    // contributions of the rows finished in earlier blocks (independent per row)
#pragma unroll
    for (int q = 0; q < blk * RB; ++q) {
      const int k = LOWER ? q : PW - 1 - q;
      const bool kin = LOWER ? true : (k < a.pw);
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        const int i = LOWER ? blk * RB + rr : PW - 1 - (blk * RB + rr);
        if (kin && i < a.pw) {
          const double ur = sre[i * SP + k], ui = sim[i * SP + k];
          ar[rr] -= ur * xr[k] - ui * xi[k];
          ai[rr] -= ur * xi[k] + ui * xr[k];
        }
      }
    }
    // in-block recurrence
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = LOWER ? blk * RB + rr : PW - 1 - (blk * RB + rr);
      double sr = ar[rr], si = ai[rr];
      if (i < a.pw) {
#pragma unroll
        for (int q = 0; q < rr; ++q) {
          const int k = LOWER ? blk * RB + q : PW - 1 - (blk * RB + q);
          if (LOWER || k < a.pw) {
            const double ur = sre[i * SP + k], ui = sim[i * SP + k];
            sr -= ur * xr[k] - ui * xi[k];
            si -= ur * xi[k] + ui * xr[k];
          }
        }
        if (!LOWER) {
          const double dr = sre[i * SP + i], di = sim[i * SP + i];
          const double den = dr * dr + di * di;
          const double qr = (sr * dr + si * di) / den, qi = (si * dr - sr * di) / den;
          sr = qr;
          si = qi;
        }
      }
      xr[i] = sr;
      xi[i] = si;
    }
  }
  double* out = LOWER ? a.linv : a.uinv;
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    out[i * PW + c] = xr[i];
    out[PW * PW + i * PW + c] = xi[i];
  }
}

// Inverse X of the unit-lower 32x32 diagonal block (rows 0..31 of the CTA's
// panel) by all PT threads in 8x8 blocks: the four diagonal blocks by forward
// substitution (one column per thread, chains of <= 7), then the off-diagonal
// blocks by distance d = 1..3, X_ij = -X_ii (sum_m L_im X_mj), one entry per
// thread -- 7 barriers instead of one warp's 32-row recurrence.  w: 64 rows of
// pitch SP of free shared memory (X in rows 0..31, the partial products T in
// rows 32..63).
__device__ void linv_blocked(const PanelArgs& a, const double* Lr, const double* Li, double* wr, double* wi) {
  constexpr int B8 = 8;
  const int tid = threadIdx.x;
  double* Tr = wr + PW * SP;
  double* Ti = wi + PW * SP;
  for (int e = tid; e < PW * PW; e += PT) {
    const int r = e / PW, c = e % PW;
    wr[r * SP + c] = 0.0;
    wi[r * SP + c] = 0.0;
  }
  __syncthreads();
  if (tid < PW) {  // diagonal blocks: column c of block b = c / 8
    const int c = tid, b0 = (c / B8) * B8;
    wr[c * SP + c] = 1.0;
    for (int r = c + 1; r < b0 + B8; ++r) {
      double sr = 0.0, si = 0.0;
      for (int k = c; k < r; ++k) {
        const double lr = Lr[r * SP + k], li = Li[r * SP + k], xr = wr[k * SP + c], xi = wi[k * SP + c];
        sr -= lr * xr - li * xi;
        si -= lr * xi + li * xr;
      }
      wr[r * SP + c] = sr;
      wi[r * SP + c] = si;
    }
  }
  __syncthreads();
  for (int d = 1; d < PW / B8; ++d) {
    const int nblk = PW / B8 - d;  // blocks (j + d, j), j < nblk
    // T = sum_{k = 8j}^{8(j+d)-1} L[r][k] X[k][c]   (r in block j+d, c in block j)
    for (int e = tid; e < nblk * B8 * B8; e += PT) {
      const int j = e / (B8 * B8), r = (j + d) * B8 + (e / B8) % B8, c = j * B8 + e % B8;
      double sr = 0.0, si = 0.0;
      for (int k = j * B8; k < (j + d) * B8; ++k) {
        const double lr = Lr[r * SP + k], li = Li[r * SP + k], xr = wr[k * SP + c], xi = wi[k * SP + c];
        sr += lr * xr - li * xi;
        si += lr * xi + li * xr;
      }
      Tr[r * SP + c] = sr;
      Ti[r * SP + c] = si;
    }
    __syncthreads();
    // X[r][c] = -sum_{k = 8(j+d)}^{r} X[r][k] T[k][c]
    for (int e = tid; e < nblk * B8 * B8; e += PT) {
      const int j = e / (B8 * B8), r = (j + d) * B8 + (e / B8) % B8, c = j * B8 + e % B8;
      double sr = 0.0, si = 0.0;
      for (int k = (j + d) * B8; k <= r; ++k) {
        const double xr = wr[r * SP + k], xi = wi[r * SP + k], tr = Tr[k * SP + c], ti = Ti[k * SP + c];
        sr -= xr * tr - xi * ti;
        si -= xr * ti + xi * tr;
      }
      wr[r * SP + c] = sr;
      wi[r * SP + c] = si;
    }
    __syncthreads();
  }
  for (int e = tid; e < PW * PW; e += PT) {
    const int r = e / PW, c = e % PW;
    a.linv[e] = wr[r * SP + c];
    a.linv[PW * PW + e] = wi[r * SP + c];
  }
}

// Write the panel back, then (CTA 0) the interchange list and the diagonal-block inverses.
__device__ void panel_finish(const PanelArgs& a, double* sre, double* sim, const int* s_piv,
                             int g, int rbeg, int cnt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < cnt * a.pw; e += PT) {
    int lr = e / a.pw, c = e % a.pw;
    long long off = (long long)(rbeg + lr) * a.ld + a.c0 + c;
    a.re[off] = sre[lr * SP + c];
    a.im[off] = sim[lr * SP + c];
  }
  if (g != 0) return;
  if (warp == 0) {
    // (dst, src) list of the panel's interchanges (dst row <- content of src row)
    const int t = lane;
    const int bend = a.c0 + a.pw;
    const int pt = t < a.pw ? s_piv[t] : -1;
    const bool extra = t < a.pw && pt >= bend;
    int first = t;
    if (extra)
      for (int q = 0; q < t; ++q)
        if (s_piv[q] == pt) { first = q; break; }
    const unsigned repmask = __ballot_sync(0xffffffffu, extra && first == t);
    const int nextra = __popc(repmask);
    const int slot = __popc(repmask & ((1u << first) - 1u));
    __shared__ int s_pos[PW], s_row[2 * PW], s_content[2 * PW];
    if (t < a.pw) s_pos[t] = extra ? a.pw + slot : pt - a.c0;
    if (t < a.pw) s_row[t] = a.c0 + t;
    if (extra && first == t) s_row[a.pw + slot] = pt;
    __syncwarp();
    const int total = a.pw + nextra;
    for (int q = t; q < total; q += 32) s_content[q] = s_row[q];
    __syncwarp();
    if (t == 0) {
      for (int q = 0; q < a.pw; ++q) {
        int x = s_content[q];
        s_content[q] = s_content[s_pos[q]];
        s_content[s_pos[q]] = x;
      }
      a.list[0] = total;
    }
    __syncwarp();
    for (int q = t; q < total; q += 32) {
      a.list[1 + q] = s_row[q];
      a.list[1 + 2 * PW + q] = s_content[q];
    }
  }
  // unit-lower inverse: blocked over the whole CTA when rows 32..95 of the
  // panel buffer are free scratch (written back above), else one warp
  if (a.pw == PW && cnt >= 3 * PW) {
    __syncthreads();
    linv_blocked(a, sre, sim, sre + PW * SP, sim + PW * SP);
  } else if (warp == 1) {
    tri_inverse<true>(a, sre, sim, lane);
  }
  // the upper-block inverses are only needed by the solves: computed for all
  // blocks at once after the factorization (uinv_batched_launch), off the
  // panel's critical path (~30 us per panel here)
}


// Inverses of the upper 32x32 diagonal blocks of a finished factorization, one
// warp per (block, item): column `lane` by back substitution, rows in blocks
// of 8 as tri_inverse.  Off the critical path (after the last panel).
__global__ void uinv_kernel(int n, const double* __restrict__ re, const double* __restrict__ im, long long ld,
                            long long slu, double* __restrict__ dinv, long long sdinv) {
  constexpr int RB = 8;
  const int lane = threadIdx.x & 31;
  const int blk = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  const int nblk = (n + PW - 1) / PW;
  if (blk >= nblk) return;
  const int c0 = blk * PW, pw = min(PW, n - c0);
  re += b * slu + (long long)c0 * ld + c0;
  im += b * slu + (long long)c0 * ld + c0;
  double* out = dinv + b * sdinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW;
  const int c = lane;
  double xr[PW], xi[PW];
#pragma unroll
  for (int bb = 0; bb < PW / RB; ++bb) {
    double ar[RB], ai[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = PW - 1 - (bb * RB + rr);
      ar[rr] = (i == c) ? 1.0 : 0.0;
      ai[rr] = 0.0;
    }
#pragma unroll
    for (int q = 0; q < bb * RB; ++q) {
      const int k = PW - 1 - q;
      if (k < pw) {
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
          const int i = PW - 1 - (bb * RB + rr);
          if (i < pw) {
            const double ur = __ldg(re + (long long)i * ld + k), ui = __ldg(im + (long long)i * ld + k);
            ar[rr] -= ur * xr[k] - ui * xi[k];
            ai[rr] -= ur * xi[k] + ui * xr[k];
          }
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = PW - 1 - (bb * RB + rr);
      double sr = ar[rr], si = ai[rr];
      if (i < pw) {
#pragma unroll
        for (int q = 0; q < rr; ++q) {
          const int k = PW - 1 - (bb * RB + q);
          if (k < pw) {
            const double ur = __ldg(re + (long long)i * ld + k), ui = __ldg(im + (long long)i * ld + k);
            sr -= ur * xr[k] - ui * xi[k];
            si -= ur * xi[k] + ui * xr[k];
          }
        }
        const double dr = __ldg(re + (long long)i * ld + i), di = __ldg(im + (long long)i * ld + i);
        const double den = dr * dr + di * di;
        const double qr = (sr * dr + si * di) / den, qi = (si * dr - sr * di) / den;
        sr = qr;
        si = qi;
      }
      xr[i] = sr;
      xi[i] = si;
    }
  }
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    out[i * PW + c] = xr[i];
    out[PW * PW + i * PW + c] = xi[i];
  }
}

}  // namespace

cudaError_t uinv_batched_launch(int n, int count, const double* re, const double* im, long long ld,
                                long long slu, double* dinv, long long sdinv, cudaStream_t st) {
  const int nblk = (n + PW - 1) / PW;
  uinv_kernel<<<dim3((nblk + 3) / 4, count), 128, 0, st>>>(n, re, im, ld, slu, dinv, sdinv);
  count_launch();
  return cudaGetLastError();
}

namespace {

// Phase timers of CTA 0 / thread 0 (read with fb_debug_panel_profile; tools/).
__device__ unsigned long long g_panel_prof[8];
__device__ unsigned long long g_panel_wall[4];  // CTA 0: sum of (globaltimer ns, clock64 cycles) over launches; [3]: sum of all-CTA spans
__device__ unsigned long long g_pstart[1024], g_pend[1024];  // per panel (item 0): first CTA start, last CTA end
[[maybe_unused]] __device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Phase probes and per-launch timing are compiled in only with
// -DFB_PANEL_PROFILE: their same-address global atomics serialise in L2 and the
// kernel cannot retire before they drain (~45 us per 32-column panel,
// tools/panel_bench.cu).
#ifdef FB_PANEL_PROFILE
#define PROBE_START long long _t_last = clock64()
#define PROBE(k)                                          \
  do {                                                    \
    if (g == 0 && tid == 0) {                             \
      long long _now = clock64();                         \
      atomicAdd(&g_panel_prof[k], (unsigned long long)(_now - _t_last)); \
      _t_last = _now;                                     \
    }                                                     \
  } while (0)
#define PROF_ONLY(x) x
#else
#define PROBE_START
#define PROBE(k) \
  do {           \
  } while (0)
#define PROF_ONLY(x)
#endif

template <int MODE>
__global__ void __launch_bounds__(PT) panel_kernel(PanelArgs a0) {
  PanelArgs a = a0;
  {
    const long long item = a.b0 + blockIdx.y;
    a.re += item * a.slu;
    a.im += item * a.slu;
    a.piv += item * a.spiv;
    a.info += item;
    a.linv += item * a.sdinv;
    a.uinv += item * a.sdinv;
    a.list += 2 * item * a.sdinv;
    a.xrec += item * a.sxs;
    a.xrowr += item * a.sxs;
    a.xu += item * a.sxs;
  }
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int G, g;
  if (MODE == PANEL_CLUSTER) {
    G = (int)cg::this_cluster().num_blocks();
    g = (int)cg::this_cluster().block_rank();
  } else {
    G = gridDim.x;
    g = blockIdx.x;
  }
  const int rbeg = a.c0 + g * a.rpc;
  const int rend = min(a.n, rbeg + a.rpc);
  const int cnt = max(0, rend - rbeg);
  double* sre = sm;                       // [rpc][SP]
  double* sim = sm + a.rpc * SP;          // [rpc][SP]
  double* prow = sim + a.rpc * SP;        // [2*PW] pivot row
  double* rrow = prow + 2 * PW;           // [2*PW] old row rj
  double* lrec = rrow + 2 * PW;           // CLUSTER: [2][REC] own record
  double* lrj = lrec + 2 * REC;           // CLUSTER: [2][2*PW] own copy of row rj
  double* mbox = lrj + 2 * 2 * PW + 4 * SB * PW;  // CLUSTER: [2][MAXG][2] pushed candidates
  __shared__ Best red[NW];
  __shared__ int s_p, s_zero;
  __shared__ int s_piv[PW];

  // panel rows -> shared memory, all loads in flight at once (cp.async)
  for (int e = tid; e < cnt * PW; e += PT) {
    int lr = e / PW, c = e % PW;
    bool ok = c < a.pw;
    long long off = ok ? (long long)(rbeg + lr) * a.ld + a.c0 + c : 0;
    cp_async8(&sre[lr * SP + c], a.re + off, ok);
    cp_async8(&sim[lr * SP + c], a.im + off, ok);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  __shared__ double s_inv[2];
  double* ubuf = lrj + 2 * 2 * PW;        // [2][SB][PW] U rows of the finished sub-block
  for (int j = 0; j < a.pw; ++j) {
    PROBE_START;
    const int rj = a.c0 + j;
    const int par = j & 1;
    const int sb0 = (j / SB) * SB, sb_end = min(a.pw, sb0 + SB);
    const bool own_rj = rj >= rbeg && rj < rend;
    // 1. local argmax of |a[r, j]| over own rows r >= rj
    Best b{-1.0, 0x7fffffff};
    for (int lr = max(0, rj - rbeg) + tid; lr < cnt; lr += PT)
      b = better(b, Best{cabs_(sre[lr * SP + j], sim[lr * SP + j]), rbeg + lr});
    b = warp_best(b);
    if (lane == 0) red[warp] = b;
    __syncthreads();
    PROBE(0);
    // 2. publish the CTA candidate (warp 0) and the current row rj (warp 1, owner)
    if (warp == 0) {
      Best t = lane < NW ? red[lane] : Best{-1.0, 0x7fffffff};
      t = warp_best(t);
      const bool own_best = t.v >= 0.0 && t.r >= rbeg && t.r < rend;
      double* rec = MODE == PANEL_CLUSTER ? lrec + par * REC : a.xrec + ((size_t)par * G + g) * REC;
      const double d0 = lane == 0 ? t.v : (double)t.r;
      const double vr = own_best ? sre[(t.r - rbeg) * SP + lane] : 0.0;
      const double vi = own_best ? sim[(t.r - rbeg) * SP + lane] : 0.0;
      if (MODE == PANEL_CLUSTER) {
        if (own_best) {
          rec[2 + lane] = vr;
          rec[2 + PW + lane] = vi;
        }
        if (lane < G) {  // push (|pivot|^2, row) into every CTA's mailbox slot g
          double* box = cg::this_cluster().map_shared_rank(mbox + (par * MAXG + g) * 2, lane);
          box[0] = t.v;
          box[1] = (double)t.r;
        }
      } else {
        if (lane < 2) __stcg(rec + lane, d0);
        if (own_best) {
          __stcg(rec + 2 + lane, vr);
          __stcg(rec + 2 + PW + lane, vi);
        }
      }
    } else if (warp == 1 && own_rj) {
      double* dst = MODE == PANEL_CLUSTER ? lrj + par * 2 * PW : a.xrowr + par * 2 * PW;
      const double vr = sre[(rj - rbeg) * SP + lane], vi = sim[(rj - rbeg) * SP + lane];
      if (MODE == PANEL_CLUSTER) {
        dst[lane] = vr;
        dst[PW + lane] = vi;
      } else {
        __stcg(dst + lane, vr);
        __stcg(dst + PW + lane, vi);
      }
    }
    PROBE(1);
    // 3. exchange barrier
    if (MODE == PANEL_CLUSTER) {
      cg::this_cluster().sync();
    } else if (G > 1) {
      __threadfence();
      cg::this_grid().sync();
    } else {
      __syncthreads();
    }
    PROBE(2);
    // 4. winner, pivot row, old row rj, pivot reciprocal (warp 0)
    if (warp == 0) {
      const int rj_owner = (rj - a.c0) / a.rpc;
      double r0, r1;  // old row rj, fetched while the candidates are reduced
      if (MODE == PANEL_CLUSTER) {
        const double* rsrc = cg::this_cluster().map_shared_rank(lrj + par * 2 * PW, rj_owner);
        r0 = rsrc[lane];
        r1 = rsrc[PW + lane];
      } else {
        r0 = __ldcg(a.xrowr + par * 2 * PW + lane);
        r1 = __ldcg(a.xrowr + par * 2 * PW + PW + lane);
      }
      Best w{-1.0, 0x7fffffff};
      int wg = 0;
      for (int q = lane; q < G; q += 32) {
        Best t;
        if (MODE == PANEL_CLUSTER) {
          const double* rr = mbox + (par * MAXG + q) * 2;
          t = Best{rr[0], (int)rr[1]};
        } else {
          const double* rr = a.xrec + ((size_t)par * G + q) * REC;
          t = Best{__ldcg(rr), (int)__ldcg(rr + 1)};
        }
        Best nb = better(w, t);
        if (nb.r != w.r || nb.v != w.v) wg = q;
        w = nb;
      }
      Best wb = warp_best(w);
      const unsigned m = __ballot_sync(0xffffffffu, w.r == wb.r && w.v == wb.v && w.v >= 0.0);
      const int gw = __shfl_sync(0xffffffffu, wg, m ? __ffs(m) - 1 : 0);
      double p0, p1;
      if (MODE == PANEL_CLUSTER) {
        const double* src = cg::this_cluster().map_shared_rank(lrec + par * REC, gw);
        p0 = src[2 + lane];
        p1 = src[2 + PW + lane];
      } else {
        const double* src = a.xrec + ((size_t)par * G + gw) * REC;
        p0 = __ldcg(src + 2 + lane);
        p1 = __ldcg(src + 2 + PW + lane);
      }
      prow[lane] = p0;
      prow[PW + lane] = p1;
      rrow[lane] = r0;
      rrow[PW + lane] = r1;
      const bool zero = !(wb.v > 0.0);
      if (lane == j) {  // lane j holds the pivot value
        double den = p0 * p0 + p1 * p1;
        s_inv[0] = zero ? 0.0 : p0 / den;
        s_inv[1] = zero ? 0.0 : -p1 / den;
      }
      if (lane == 0) {
        const int p = zero ? rj : wb.r;
        s_p = p;
        s_zero = zero;
        s_piv[j] = p;
        if (g == 0) {
          a.piv[rj] = p;
          if (zero) atomicMin(a.info, rj + 1);
        }
      }
    }
    __syncthreads();
    PROBE(3);
    const int p = s_p;
    const bool zero = s_zero;
    // 5. full-row swap (one warp per moved row, lanes over columns)
    if (p != rj) {
      if (warp == 2 && p >= rbeg && p < rend) {
        sre[(p - rbeg) * SP + lane] = rrow[lane];
        sim[(p - rbeg) * SP + lane] = rrow[PW + lane];
      } else if (warp == 3 && own_rj) {
        sre[(rj - rbeg) * SP + lane] = prow[lane];
        sim[(rj - rbeg) * SP + lane] = prow[PW + lane];
      }
      __syncthreads();
    }
    PROBE(4);
    // 6. multipliers and the rank-1 update inside the current sub-block only
    if (!zero) {
      const double ir = s_inv[0], ii = s_inv[1];
      for (int lr = max(0, rj + 1 - rbeg) + tid; lr < cnt; lr += PT) {
        const double xr = sre[lr * SP + j], xi = sim[lr * SP + j];
        const double lre = xr * ir - xi * ii, lim = xr * ii + xi * ir;
        sre[lr * SP + j] = lre;
        sim[lr * SP + j] = lim;
        for (int c = j + 1; c < sb_end; ++c) {
          const double ur = prow[c], ui = prow[PW + c];
          sre[lr * SP + c] -= lre * ur - lim * ui;
          sim[lr * SP + c] -= lre * ui + lim * ur;
        }
      }
    }
    __syncthreads();
    // 7. end of a sub-block: U rows of the sub-block for the remaining panel
    //    columns (CTA 0, forward substitution with the unit-lower block), then
    //    A[r, rest] -= L[r, sub] U[sub, rest] for every row below the sub-block.
    if (j == sb_end - 1 && sb_end < a.pw) {
      const int rest = a.pw - sb_end, nsub = sb_end - sb0;
      if (g == 0) {
        if (tid < rest) {
          const int c = sb_end + tid;
          for (int i = 1; i < nsub; ++i) {
            double ar = sre[(sb0 + i) * SP + c], ai = sim[(sb0 + i) * SP + c];
            for (int k = 0; k < i; ++k) {
              const double lr_ = sre[(sb0 + i) * SP + sb0 + k], li = sim[(sb0 + i) * SP + sb0 + k];
              const double ur = sre[(sb0 + k) * SP + c], ui = sim[(sb0 + k) * SP + c];
              ar -= lr_ * ur - li * ui;
              ai -= lr_ * ui + li * ur;
            }
            sre[(sb0 + i) * SP + c] = ar;
            sim[(sb0 + i) * SP + c] = ai;
          }
        }
        __syncthreads();
        double* ub = ubuf + par * 2 * SB * PW;  // [2 planes][SB][PW]
        for (int e = tid; e < nsub * PW; e += PT) {
          const int i = e / PW, c = e % PW;
          const double vr = sre[(sb0 + i) * SP + c], vi = sim[(sb0 + i) * SP + c];
          if (MODE == PANEL_CLUSTER) {
            ub[i * PW + c] = vr;
            ub[SB * PW + i * PW + c] = vi;
          } else {
            __stcg(a.xu + par * 2 * SB * PW + i * PW + c, vr);
            __stcg(a.xu + par * 2 * SB * PW + SB * PW + i * PW + c, vi);
          }
        }
      }
      if (MODE == PANEL_CLUSTER) {
        cg::this_cluster().sync();
      } else if (G > 1) {
        __threadfence();
        cg::this_grid().sync();
      } else {
        __syncthreads();
      }
      // fetch U[sub, rest] into prow/rrow-free scratch (reuse the record area of parity par^1)
      double* uloc = ubuf + (par ^ 1) * 2 * SB * PW;
      if (g != 0 || MODE != PANEL_CLUSTER) {
        for (int e = tid; e < nsub * PW; e += PT) {
          double vr, vi;
          if (MODE == PANEL_CLUSTER) {
            const double* src = cg::this_cluster().map_shared_rank(ubuf + par * 2 * SB * PW, 0);
            vr = src[e];
            vi = src[SB * PW + e];
          } else {
            vr = __ldcg(a.xu + par * 2 * SB * PW + e);
            vi = __ldcg(a.xu + par * 2 * SB * PW + SB * PW + e);
          }
          uloc[e] = vr;
          uloc[SB * PW + e] = vi;
        }
      } else {
        for (int e = tid; e < nsub * PW; e += PT) {
          uloc[e] = ubuf[par * 2 * SB * PW + e];
          uloc[SB * PW + e] = ubuf[par * 2 * SB * PW + SB * PW + e];
        }
      }
      __syncthreads();
      for (int lr = max(0, a.c0 + sb_end - rbeg) + tid; lr < cnt; lr += PT) {
        for (int c = sb_end; c < a.pw; ++c) {
          double ar = sre[lr * SP + c], ai = sim[lr * SP + c];
          for (int k = 0; k < nsub; ++k) {
            const double lr_ = sre[lr * SP + sb0 + k], li = sim[lr * SP + sb0 + k];
            const double ur = uloc[k * PW + c], ui = uloc[SB * PW + k * PW + c];
            ar -= lr_ * ur - li * ui;
            ai -= lr_ * ui + li * ur;
          }
          sre[lr * SP + c] = ar;
          sim[lr * SP + c] = ai;
        }
      }
      __syncthreads();
    }
    PROBE(5);
  }
  if (MODE == PANEL_CLUSTER) cg::this_cluster().sync();  // remote readers done before exit

  panel_finish(a, sre, sim, s_piv, g, rbeg, cnt);
}

// Cluster path: every row of the panel is owned by one thread of one CTA for
// the whole factorization, and every CTA PUSHES its column candidate (|pivot|^2,
// row, full panel row) and, if it owns it, the current row rj into the
// mailboxes of all CTAs before the cluster barrier.  After the barrier each
// thread reduces the (local) mailbox itself, so a column costs one
// __syncthreads, one barrier.cluster and no remote reads.
__global__ void __launch_bounds__(PT) panel_cluster_kernel(PanelArgs a0) {
  if (a0.pw < 0) return;  // launch-cost probe (tools/panel_bench.cu)
  PanelArgs a = a0;
  {
    const long long item = a.b0 + blockIdx.y;
    a.re += item * a.slu;
    a.im += item * a.slu;
    a.piv += item * a.spiv;
    a.info += item;
    a.linv += item * a.sdinv;
    a.uinv += item * a.sdinv;
    a.list += 2 * item * a.sdinv;
    a.xrec += item * a.sxs;
    a.xrowr += item * a.sxs;
    a.xu += item * a.sxs;
  }
  PROF_ONLY(const long long _t_kernel0 = clock64(); const unsigned long long _g_kernel0 = gtimer();
            if (threadIdx.x == 0 && blockIdx.y == 0 && a.b0 == 0 && a.c0 / PW < 1024)
                atomicMin(&g_pstart[a.c0 / PW], _g_kernel0);)
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = (int)cl.num_blocks(), g = (int)cl.block_rank();
  const int rbeg = a.c0 + g * a.rpc;
  const int rend = min(a.n, rbeg + a.rpc);
  const int cnt = max(0, rend - rbeg);
  double* sre = sm;                                // [rpc][SP]
  double* sim = sre + a.rpc * SP;                  // [rpc][SP]
  double* mrec = sim + a.rpc * SP;                 // [2][MAXG][REC] pushed candidates
  double* mrj = mrec + 2 * MAXG * REC;             // [2][2*PW] pushed row rj
  double* ubuf = mrj + 2 * 2 * PW;                 // [2*SB*PW] U rows of a finished sub-block
  __shared__ Best red[NW];
  __shared__ int s_piv[PW];
  __shared__ __align__(8) unsigned long long mbar[2];  // per-parity mailbox completion
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  cl.sync();  // peers may push only after our mbarriers exist

  // panel rows -> shared memory, all loads in flight at once (cp.async)
  for (int e = tid; e < cnt * PW; e += PT) {
    int lr = e / PW, c = e % PW;
    bool ok = c < a.pw;
    long long off = ok ? (long long)(rbeg + lr) * a.ld + a.c0 + c : 0;
    cp_async8(&sre[lr * SP + c], a.re + off, ok);
    cp_async8(&sim[lr * SP + c], a.im + off, ok);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  PROF_ONLY(if (g == 0 && tid == 0) atomicAdd(&g_panel_prof[6], (unsigned long long)(clock64() - _t_kernel0));)

  for (int j = 0; j < a.pw; ++j) {
    PROBE_START;
    const int rj = a.c0 + j;
    const int par = j & 1;
    const int sb0 = (j / SB) * SB, sb_end = min(a.pw, sb0 + SB);
    const bool own_rj = rj >= rbeg && rj < rend;
    // 1. argmax of |a(r, j)|^2 over own rows r >= rj
    Best b{-1.0, 0x7fffffff};
    for (int lr = tid; lr < cnt; lr += PT) {  // own rows only (no barrier since step 4)
      if (rbeg + lr < rj) continue;
      b = better(b, Best{cabs_(sre[lr * SP + j], sim[lr * SP + j]), rbeg + lr});
    }
    b = warp_best(b);
    if (lane == 0) red[warp] = b;
    __syncthreads();
    PROBE(0);
    // 2. CTA candidate (every warp reduces red[]); warp w pushes it (st.async)
    //    into the mailboxes of CTAs w, w+NW, ...; the owner of row rj pushes it too.
    //    Each CTA expects G records + one row rj per column on mbar[par].
    {
      if (tid == 0) mbar_arrive_expect_tx(&mbar[par], (unsigned)(G * REC * 8 + 2 * PW * 8));
      Best t = lane < NW ? red[lane] : Best{-1.0, 0x7fffffff};
      t = warp_best(t);
      const bool has = t.v >= 0.0;
      const int lr = has ? t.r - rbeg : 0;
      // pair l of the record: l = 0 -> (|pivot|, row); l = 1..16 -> re[2l-2..]; 17..32 -> im
      const int rb = 2 * lane;  // this lane's data pair covers columns rb, rb+1 of re (lane<16) or im
      double x0, x1;
      if (lane < 16) {
        x0 = has ? sre[lr * SP + rb] : 0.0;
        x1 = has ? sre[lr * SP + rb + 1] : 0.0;
      } else {
        x0 = has ? sim[lr * SP + rb - PW] : 0.0;
        x1 = has ? sim[lr * SP + rb - PW + 1] : 0.0;
      }
      double w0 = 0.0, w1 = 0.0;
      if (own_rj) {
        const int l2 = rj - rbeg;
        if (lane < 16) {
          w0 = sre[l2 * SP + rb];
          w1 = sre[l2 * SP + rb + 1];
        } else {
          w0 = sim[l2 * SP + rb - PW];
          w1 = sim[l2 * SP + rb - PW + 1];
        }
      }
      const unsigned rec_l = smem_u32(mrec + (par * MAXG + g) * REC);
      const unsigned rj_l = smem_u32(mrj + par * 2 * PW);
      const unsigned bar_l = smem_u32(&mbar[par]);
      for (int q = warp; q < G; q += NW) {
        const unsigned rrec = mapa_u32(rec_l, q), rbar = mapa_u32(bar_l, q);
        st_async_v2(rrec + 16 + 16 * lane, x0, x1, rbar);
        if (lane == 0) st_async_v2(rrec, t.v, __longlong_as_double((long long)t.r), rbar);  // row as integer bits
        if (own_rj) st_async_v2(mapa_u32(rj_l, q) + 16 * lane, w0, w1, rbar);
      }
    }
    PROBE(1);
    mbar_wait_parity(&mbar[par], (j >> 1) & 1);
    PROBE(2);
    // 3. winner from the local mailbox (every warp, redundantly)
    const double* rec = mrec + par * MAXG * REC;
    Best w = lane < G ? Best{rec[lane * REC], (int)__double_as_longlong(rec[lane * REC + 1])}
                      : Best{-1.0, 0x7fffffff};
    const Best wb = warp_best(w);
    const unsigned m = __ballot_sync(0xffffffffu, lane < G && w.r == wb.r && w.v == wb.v);
    const int gw = m ? __ffs(m) - 1 : 0;
    const bool zero = !(wb.v > 0.0);
    const int p = zero ? rj : wb.r;
    const double* prow = rec + gw * REC + 2;     // pivot row (re[PW], im[PW])
    const double* rrow = mrj + par * 2 * PW;      // old row rj
    if (tid == 0) {
      s_piv[j] = p;
      if (g == 0) {
        a.piv[rj] = p;
        if (zero) atomicMin(a.info, rj + 1);
      }
    }
    double ir = 0.0, ii = 0.0;
    if (!zero) {
      const double pr = prow[j], pi = prow[PW + j];
      const double den = pr * pr + pi * pi;
      const double rden = 1.0 / den;  // one division on the critical path
      ir = pr * rden;
      ii = -pi * rden;
    }
    PROBE(3);
    // 4. own rows: swap (by the owning warp, lanes over columns), multiplier,
    //    rank-1 update inside the sub-block
    if (p != rj) {
      if (own_rj && (((rj - rbeg) % PT) >> 5) == warp) {
        sre[(rj - rbeg) * SP + lane] = prow[lane];
        sim[(rj - rbeg) * SP + lane] = prow[PW + lane];
      }
      if (p >= rbeg && p < rend && (((p - rbeg) % PT) >> 5) == warp) {
        sre[(p - rbeg) * SP + lane] = rrow[lane];
        sim[(p - rbeg) * SP + lane] = rrow[PW + lane];
      }
      __syncwarp();
    }
    for (int lr = tid; lr < cnt; lr += PT) {
      const int gr = rbeg + lr;
      if (gr <= rj || zero) continue;
      const double xr = sre[lr * SP + j], xi = sim[lr * SP + j];
      const double lre = xr * ir - xi * ii, lim = xr * ii + xi * ir;
      sre[lr * SP + j] = lre;
      sim[lr * SP + j] = lim;
      for (int c = j + 1; c < sb_end; ++c) {
        const double ur = prow[c], ui = prow[PW + c];
        sre[lr * SP + c] -= lre * ur - lim * ui;
        sim[lr * SP + c] -= lre * ui + lim * ur;
      }
    }
    PROBE(4);
    // 5. end of a sub-block: U rows (CTA 0, forward substitution), pushed to all
    //    CTAs; then A[r, rest] -= L[r, sub] U[sub, rest] on the rows below.
    if (j == sb_end - 1 && sb_end < a.pw) {
      const int rest = a.pw - sb_end, nsub = sb_end - sb0;
      __syncthreads();
      if (g == 0) {
        if (tid < rest) {
          const int c = sb_end + tid;
          for (int i = 1; i < nsub; ++i) {
            double ar = sre[(sb0 + i) * SP + c], ai = sim[(sb0 + i) * SP + c];
            for (int k = 0; k < i; ++k) {
              const double lr_ = sre[(sb0 + i) * SP + sb0 + k], li = sim[(sb0 + i) * SP + sb0 + k];
              const double ur = sre[(sb0 + k) * SP + c], ui = sim[(sb0 + k) * SP + c];
              ar -= lr_ * ur - li * ui;
              ai -= lr_ * ui + li * ur;
            }
            sre[(sb0 + i) * SP + c] = ar;
            sim[(sb0 + i) * SP + c] = ai;
          }
        }
        __syncthreads();
        for (int e = tid; e < G * nsub * PW; e += PT) {
          const int q = e / (nsub * PW), f = e % (nsub * PW), i = f / PW, c = f % PW;
          double* ub = cl.map_shared_rank(ubuf, q);
          ub[i * PW + c] = sre[(sb0 + i) * SP + c];
          ub[SB * PW + i * PW + c] = sim[(sb0 + i) * SP + c];
        }
      }
      cl.sync();
      for (int lr = max(0, a.c0 + sb_end - rbeg) + tid; lr < cnt; lr += PT) {
        for (int c = sb_end; c < a.pw; ++c) {
          double ar = sre[lr * SP + c], ai = sim[lr * SP + c];
          for (int k = 0; k < nsub; ++k) {
            const double lr_ = sre[lr * SP + sb0 + k], li = sim[lr * SP + sb0 + k];
            const double ur = ubuf[k * PW + c], ui = ubuf[SB * PW + k * PW + c];
            ar -= lr_ * ur - li * ui;
            ai -= lr_ * ui + li * ur;
          }
          sre[lr * SP + c] = ar;
          sim[lr * SP + c] = ai;
        }
      }
      cl.sync();  // ubuf is rewritten by CTA 0 at the next sub-block end
    }
    PROBE(5);
  }
  cl.sync();  // remote writers done before anyone exits
  __syncthreads();

  PROF_ONLY(const long long _t_fin0 = clock64();)
  panel_finish(a, sre, sim, s_piv, g, rbeg, cnt);
  PROF_ONLY(if (tid == 0 && blockIdx.y == 0 && a.b0 == 0 && a.c0 / PW < 1024) atomicMax(&g_pend[a.c0 / PW], gtimer());
            if (g == 0 && tid == 0) {
              atomicAdd(&g_panel_prof[7], (unsigned long long)(clock64() - _t_fin0));
              atomicAdd(&g_panel_wall[0], gtimer() - _g_kernel0);
              atomicAdd(&g_panel_wall[1], (unsigned long long)(clock64() - _t_kernel0));
              atomicAdd(&g_panel_wall[2], 1ull);
            })
}

size_t panel_cluster_smem(int rpc) {
  return sizeof(double) * (2 * (size_t)rpc * SP + 2 * MAXG * REC + 4 * PW + 2 * SB * PW);
}

int g_grid_max_blocks = 0;
bool g_cluster_ok = false;

size_t panel_smem(int rpc) {
  return sizeof(double) * (2 * (size_t)rpc * SP + 4 * PW + 2 * REC + 4 * PW + 4 * SB * PW + 4 * MAXG);
}

}  // namespace

void panel_span_raw(unsigned long long* s0, unsigned long long* e0) {
  cudaMemcpyFromSymbol(s0, g_pstart, 8);
  cudaMemcpyFromSymbol(e0, g_pend, 8);
}

void panel_wall_read(unsigned long long* out4) {
  static unsigned long long st[1024], en[1024];
  cudaMemcpyFromSymbol(st, g_pstart, sizeof(st));
  cudaMemcpyFromSymbol(en, g_pend, sizeof(en));
  cudaMemcpyFromSymbol(out4, g_panel_wall, sizeof(unsigned long long) * 4);
  unsigned long long sum = 0;
  for (int i = 0; i < 1024; ++i)
    if (en[i] > st[i] && st[i] != ~0ull) sum += en[i] - st[i];
  out4[3] = sum;   // sum over panels of (last CTA end - first CTA start), item 0
  for (int i = 0; i < 1024; ++i) {
    st[i] = ~0ull;
    en[i] = 0ull;
  }
  cudaMemcpyToSymbol(g_pstart, st, sizeof(st));
  cudaMemcpyToSymbol(g_pend, en, sizeof(en));
  unsigned long long z[4] = {0};
  cudaMemcpyToSymbol(g_panel_wall, z, sizeof(z));
}

void panel_profile_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_panel_prof, sizeof(unsigned long long) * 8);
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_panel_prof, z, sizeof(z));
}

size_t panel_scratch_bytes() {
  const int Gmax = 4 * kSMs;
  return sizeof(double) * (2 * (size_t)Gmax * REC + 2 * 2 * PW + 4 * SB * PW) + 256;
}

cudaError_t panel_launch(PanelArgs a, int count, char* scratch, cudaStream_t st) {
  const int rows = a.n - a.c0;
  const int smem_cap = 226 * 1024;  // 227 KB opt-in minus the kernels' static shared memory
  const int rpc_cluster = 384;
  const int max_cluster = 16;
  double* d = reinterpret_cast<double*>(scratch);
  const int Gmax = 4 * kSMs;
  a.xrec = d;
  a.xrowr = d + 2 * (size_t)Gmax * REC;
  a.xu = a.xrowr + 2 * 2 * PW;
  a.sxs = (long long)(panel_scratch_bytes() / sizeof(double));
  a.b0 = 0;
  static DevOnce probed;  // attributes are per device; the probe results are the same on every B200
  if (probed.first()) {
    cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap);
    cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(panel_kernel<PANEL_GRID>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = max_cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(max_cluster);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = panel_cluster_smem(rpc_cluster);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, panel_cluster_kernel, &cfg);
    g_cluster_ok = (e == cudaSuccess && clusters >= 1);
    cudaGetLastError();
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, panel_kernel<PANEL_GRID>, PT, panel_smem(128));
    g_grid_max_blocks = std::max(1, nb);
  }
  count_launch();
  if (rows <= rpc_cluster || (g_cluster_ok && rows <= max_cluster * rpc_cluster)) {
    int G = std::max(1, std::min(max_cluster, ceil_div(rows, rpc_cluster)));
    // rows per CTA: a batch of shifts leaves the SMs to the concurrent trailing
    // GEMMs (384: fewest CTAs, +1-3 % at 8 shifts); a lone shift is panel-latency
    // bound and wants the shortest per-CTA column work (192: 28.2 vs 31.1 ms
    // for one N = 4096 LU)
    const int rmin = count >= 4 ? 384 : 192;
    if (rows > 2 * PW) G = std::max(G, std::min(max_cluster, ceil_div(rows, rmin)));
    G = std::max(1, std::min(G, rows / PW));
    int rpc = ceil_div(rows, G);
    G = ceil_div(rows, rpc);
    a.rpc = rpc;
    // G == 1 runs the cluster kernel too (a 1-CTA cluster): its exchange stays
    // in shared memory, where the grid kernel would round-trip through L2
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(G, count);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = panel_cluster_smem(rpc);
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, panel_cluster_kernel, a);
  }
  int G = ceil_div(rows, 128);
  G = std::max(1, std::min(G, rows / PW));
  G = std::min(G, g_grid_max_blocks * kSMs);
  int rpc = ceil_div(rows, G);
  G = ceil_div(rows, rpc);
  a.rpc = rpc;
  size_t smem = panel_smem(rpc);
  if ((int)smem > smem_cap) return cudaErrorInvalidConfiguration;
  // cooperative launches need every CTA co-resident: split the batch if needed
  const int per = std::max(1, (g_grid_max_blocks * kSMs) / G);
  for (int b0 = 0; b0 < count; b0 += per) {
    a.b0 = b0;
    void* args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)panel_kernel<PANEL_GRID>, dim3(G, std::min(per, count - b0)),
                                                dim3(PT), args, smem, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fb
