// Partitioned (SPIKE) shifted band LU and multi-RHS solve (banded.py:68-146,
// 156-164), batched over contour shifts.
//
// S = z*FB - FA (n x n, kl sub- and super-diagonals) is cut into P row/column
// partitions.  With A_j the diagonal blocks, B_j / C_j the kl x kl couplings
// to the next / previous partition,
//     S = diag(A_j) * (I + spikes),  V_j = A_j^-1 [0; B_j],  W_j = A_j^-1 [C_j; 0].
// Factor (once per shift):
//   pfactor   every partition's band LU with partial pivoting inside the
//             partition (dgbtf2 scheme, kv = 2kl), one warp per partition,
//             the active (kl+1) x (2kl+1) window in shared memory;
//   spikes    V_j, W_j by the partition solve with the 2kl coupling columns;
//   rfactor   the interface system (unknowns y_i = (x_i^bottom, x_{i+1}^top),
//             block tridiagonal with 2kl x 2kl blocks) by block LU; the pivot
//             blocks are inverted by Gauss-Jordan with partial pivoting.
// Solve (per contour pass):
//   psolve    g = A_j^-1 f_j for every partition (one warp per partition and
//             32 right-hand sides, lanes = columns, register windows);
//   rsolve    interface values from the block LU (one CTA per shift and chunk);
//   correct   x_j = g_j - V_j x_{j+1}^top - W_j x_{j-1}^bottom.
// Every partition block of z*B - A is nonsingular for Im z != 0 (B HPD), so
// pivoting inside partitions is enough.  The partitioned pivot order differs
// from the reference's whole-band LU; results agree to rounding.
//
// Factor storage (per shift) is the reference's working array, COLUMN-major,
// W[j*(3kl+1) + kv + i - j] = LU(i, j) (banded.py:68-103), pivots ipiv[j]
// (global row index, inside the partition).  aux (per shift):
//   spikes  [n][2kl] re | [n][2kl] im   (columns 0..kl-1: V, kl..2kl-1: W)
//   Dinv    [P-1][2kl][2kl] re | im      inverse pivot blocks of the interface LU
//   F       [P-1][kl][2kl] re | im       multipliers (top kl rows)
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "band.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "misc.cuh"

namespace fb {

namespace {

constexpr int KLMAX = 16;
constexpr int WPB = 4;  // warps per CTA in the per-partition kernels
constexpr int WIN = (KLMAX + 1) * (2 * KLMAX + 1);

struct Zs {
  double r[64], i[64];
};

// Partitions of equal size sz = ceil(n / P) (the last one shorter; P is chosen
// so that it still holds > 2kl rows): equal strides let the spike correction
// run as one strided-batch ZGEMM over the partitions.
__host__ __device__ __forceinline__ int part_sz(int n, int P) { return (n + P - 1) / P; }
__host__ __device__ __forceinline__ int part_lo(int j, int n, int P) {
  return (int)min((long long)n, (long long)j * part_sz(n, P));
}

// S[r][c] of z*FB - FA inside partition [lo, hi) (zero outside it or the band),
// with the rounding of band_shift_kernel (numpy order, banded.py:158-163)
__device__ __forceinline__ void s_entry(int r, int c, int lo, int hi, int kl, double zr, double zi,
                                        const double* far_, const double* fai, const double* fbr,
                                        const double* fbi, long long ldb, double& vr, double& vi) {
  vr = 0.0;
  vi = 0.0;
  const int s = r - c;
  if (r < lo || r >= hi || c < lo || c >= hi || s > kl || s < -kl) return;
  const long long o = (long long)(kl + s) * ldb + c;
  const double ar = far_[o], ai = fai ? fai[o] : 0.0;
  if (fbr) {
    const double br = fbr[o], bi = fbi ? fbi[o] : 0.0;
    const double pr = __dsub_rn(__dmul_rn(zr, br), __dmul_rn(zi, bi));
    const double pi = __dadd_rn(__dmul_rn(zr, bi), __dmul_rn(zi, br));
    vr = (0.0 - ar) + pr;
    vi = (0.0 - ai) + pi;
  } else {
    vr = s == 0 ? (0.0 - ar) + zr : (0.0 - ar);
    vi = s == 0 ? (0.0 - ai) + zi : (0.0 - ai);
  }
}

struct PFArgs {
  int n, kl, P;
  Zs z;
  const double *far_, *fai, *fbr, *fbi;
  long long ldb;
  double *wr, *wi;
  long long sw;  // factor batch stride (doubles)
  int* ipiv;
  long long sp;
  int* info;  // [count], INT_MAX = ok, else 1 + first zero-pivot column
};

// ---- partition band LU: one warp per (partition, shift) ------------------------
__global__ void __launch_bounds__(WPB * 32) band_pfactor_kernel(PFArgs a) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int part = blockIdx.x * WPB + wid, k = blockIdx.y;
  if (part >= a.P) return;
  const int kl = a.kl, kv = 2 * kl, LW = 3 * kl + 1, RW = kl + 1, CW = 2 * kl + 1;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  __shared__ double swin[WPB][2][WIN];
  double* xr = swin[wid][0];  // window, column-major by slot: x[cslot * RW + rslot]
  double* xi = swin[wid][1];
  double* Wr = a.wr + k * a.sw;
  double* Wi = a.wi + k * a.sw;
  int* ipiv = a.ipiv + k * a.sp;
  const double zr = a.z.r[k], zi = a.z.i[k];
  auto S = [&](int r, int c, double& vr, double& vi) {
    s_entry(r, c, lo, hi, kl, zr, zi, a.far_, a.fai, a.fbr, a.fbi, a.ldb, vr, vi);
  };
  for (int e = lane; e < RW * CW; e += 32) {
    const int ri = e % RW, ci = e / RW;
    double vr, vi;
    S(lo + ri, lo + ci, vr, vi);
    xr[ci * RW + ri] = vr;
    xi[ci * RW + ri] = vi;
  }
  int rb = 0, cb = 0;  // slots of row j / column j
  int ju = lo, bad = 0;
  // Entries entering the window at step j (row j+RW at columns j+1+c, column
  // j+CW at rows j+1+i) depend only on A, B and z: they are fetched QF steps
  // ahead into a register queue so the global latency is off the column chain.
  constexpr int QF = 4;
  struct Ent {
    double r0, i0, r1, i1, cr, ci;
  };
  auto fetch = [&](int jj) {
    Ent e{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (lane < CW) S(jj + RW, jj + 1 + lane, e.r0, e.i0);
    if (lane + 32 < CW) S(jj + RW, jj + 1 + lane + 32, e.r1, e.i1);
    if (lane < kl) S(jj + 1 + lane, jj + CW, e.cr, e.ci);
    return e;
  };
  Ent q[QF];
#pragma unroll
  for (int d = 0; d < QF; ++d) q[d] = fetch(lo + d);
  for (int j = lo; j < hi; ++j) {
    const Ent nxt = fetch(j + QF);
    __syncwarp();
    const int km = min(kl, hi - 1 - j);
    auto RS = [&](int i) { const int s = rb + i; return s >= RW ? s - RW : s; };
    auto CS = [&](int c) { const int s = cb + c; return s >= CW ? s - CW : s; };
    const int c0 = CS(0) * RW;
    // pivot: first row of max |.| among j..j+km (banded.py:79-84)
    double best = -1.0;
    int bi = 0;
    if (lane <= km) {
      best = hypot(xr[c0 + RS(lane)], xi[c0 + RS(lane)]);
      bi = lane;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    int jp = bi;
    if (!(best > 0.0)) {
      if (!bad) bad = j + 1;
      jp = 0;
    }
    if (lane == 0) ipiv[j] = j + jp;
    ju = max(ju, min(j + kl + jp, hi - 1));
    if (jp) {
      const int sa = RS(0), sb = RS(jp);
      for (int c = lane; c <= ju - j; c += 32) {
        const int cs = CS(c) * RW;
        double t = xr[cs + sa];
        xr[cs + sa] = xr[cs + sb];
        xr[cs + sb] = t;
        t = xi[cs + sa];
        xi[cs + sa] = xi[cs + sb];
        xi[cs + sb] = t;
      }
    }
    __syncwarp();
    const double pr = xr[c0 + RS(0)], pim = xi[c0 + RS(0)];
    const bool zero = !(pr != 0.0 || pim != 0.0);
    if (km > 0 && !zero) {
      const double den = pr * pr + pim * pim;
      const double ir = pr / den, ii = -pim / den;
      if (lane < km) {
        const int s = c0 + RS(1 + lane);
        const double x_r = xr[s], x_i = xi[s];
        xr[s] = x_r * ir - x_i * ii;
        xi[s] = x_r * ii + x_i * ir;
      }
      __syncwarp();
      for (int c = lane; c < ju - j; c += 32) {  // column j+1+c -= l * u
        const int cs = CS(1 + c) * RW;
        const double ur = xr[cs + RS(0)], ui = xi[cs + RS(0)];
        if (ur == 0.0 && ui == 0.0) continue;
        for (int i = 0; i < km; ++i) {
          const int s = RS(1 + i);
          const double lr = xr[c0 + s], li = xi[c0 + s];
          xr[cs + s] -= lr * ur - li * ui;
          xi[cs + s] -= lr * ui + li * ur;
        }
      }
    }
    __syncwarp();
    // row j of U (columns j..j+kv) and the multipliers of column j leave the window
    for (int c = lane; c <= kv; c += 32) {
      if (j + c < hi) {
        const long long o = (long long)(j + c) * LW + kv - c;
        Wr[o] = xr[CS(c) * RW + RS(0)];
        Wi[o] = xi[CS(c) * RW + RS(0)];
      }
    }
    if (lane < kl) {
      const long long o = (long long)j * LW + kv + 1 + lane;
      Wr[o] = lane < km ? xr[c0 + RS(1 + lane)] : 0.0;
      Wi[o] = lane < km ? xi[c0 + RS(1 + lane)] : 0.0;
    }
    __syncwarp();
    // slide: row j+kl+1 takes row j's slot, column j+2kl+1 takes column j's slot
    for (int c = lane; c < CW; c += 32) {
      const int cs = CS(1 + c) * RW;  // c = kv wraps onto column j's slot (= column j+CW)
      xr[cs + RS(0)] = c < 32 ? q[0].r0 : q[0].r1;
      xi[cs + RS(0)] = c < 32 ? q[0].i0 : q[0].i1;
    }
    if (lane < kl) {
      xr[c0 + RS(1 + lane)] = q[0].cr;
      xi[c0 + RS(1 + lane)] = q[0].ci;
    }
#pragma unroll
    for (int d = 0; d + 1 < QF; ++d) q[d] = q[d + 1];
    q[QF - 1] = nxt;
    rb = RS(1);
    cb = CS(1);
  }
  if (bad && lane == 0) atomicMin(a.info + k, bad);
}

// ---- partition solve arguments (staged sweeps below) ----------------------------
struct PSArgs {
  int n, kl, P, nrhs, count;
  const double *wr, *wi;
  long long sw;
  const int* ipiv;
  long long sp;
  const double2* us;  // slot-ordered U columns of item 0 (item k at + k*sa doubles)
  const double* t4;   // kl = 16: U in 4-row DMMA fragment order (band_t4_kernel), else nullptr
  long long sa;
  double *xr, *xi;
  long long ldx, sx;
  // forward sweep input (nullptr: in place from x); fi == nullptr: real input;
  // sf = 0: one right-hand-side block shared by every item (the pass's Y)
  const double *fr, *fi;
  long long ldf, sf;
};

// ---- spike right-hand sides: [0; B_j] in columns 0..kl-1, [C_j; 0] in kl..2kl-1 ----
struct SIArgs {
  int n, kl, P;
  Zs z;
  const double *far_, *fai, *fbr, *fbi;
  long long ldb;
  double *sr, *si;  // spike buffers [n][2kl]
  long long ss;
};

__global__ void band_spike_init_kernel(SIArgs a) {
  const int k = blockIdx.y, kl = a.kl, w = 2 * kl;
  double* Sr = a.sr + k * a.ss;
  double* Si = a.si + k * a.ss;
  const double zr = a.z.r[k], zi = a.z.i[k];
  const long long total = (long long)a.n * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / w), c = (int)(e % w);
    // partition of row r
    int j = (int)(((long long)r * a.P) / a.n);
    while (j + 1 < a.P && part_lo(j + 1, a.n, a.P) <= r) ++j;
    while (part_lo(j, a.n, a.P) > r) --j;
    const int lo = part_lo(j, a.n, a.P), hi = part_lo(j + 1, a.n, a.P);
    double vr = 0.0, vi = 0.0;
    if (c < kl) {  // B_j: rows hi-kl..hi-1, columns hi..hi+kl-1 of S
      if (j + 1 < a.P && r >= hi - kl) {
        const int nhi = part_lo(j + 2, a.n, a.P);
        s_entry(r, hi + c, 0, nhi, kl, zr, zi, a.far_, a.fai, a.fbr, a.fbi, a.ldb, vr, vi);
      }
    } else {  // C_j: rows lo..lo+kl-1, columns lo-kl..lo-1 of S
      if (j > 0 && r < lo + kl) {
        s_entry(r, lo - kl + (c - kl), 0, hi, kl, zr, zi, a.far_, a.fai, a.fbr, a.fbi, a.ldb, vr, vi);
      }
    }
    Sr[e] = vr;
    Si[e] = vi;
  }
}

// ---- interface system: block LU, one CTA per shift ------------------------------
// Block row i (interface between partitions i and i+1), unknowns y_i =
// (x_i^b, x_{i+1}^t):  D_i = [[I, V_i^b], [W_{i+1}^t, I]],
// L_i = [[W_i^b, 0], [0, 0]] (on y_{i-1}), U_i = [[0, 0], [0, V_{i+1}^t]] (on y_{i+1}).
// D'_0 = D_0, F_i = L_i D'_{i-1}^-1 (top kl rows), D'_i = D_i - F_i U_{i-1}.
struct RFArgs {
  int n, kl, P;
  const double *sr, *si;
  long long ss;
  double *dr, *di;  // Dinv [P-1][2kl][2kl]
  double *fr, *fi;  // F    [P-1][kl][2kl]
  long long sa;     // aux batch stride
  int* info;
};

constexpr int RT = 256;
constexpr int M2 = 2 * KLMAX;  // 32

__global__ void __launch_bounds__(RT) band_rfactor_kernel(RFArgs a) {
  const int k = blockIdx.x, kl = a.kl, w = 2 * kl, tid = threadIdx.x;
  const double* Sr = a.sr + k * a.ss;
  const double* Si = a.si + k * a.ss;
  double* Dr = a.dr + k * a.sa;
  double* Di = a.di + k * a.sa;
  double* Fr = a.fr + k * a.sa;
  double* Fi = a.fi + k * a.sa;
  __shared__ double ar[M2][2 * M2 + 1], ai[M2][2 * M2 + 1];  // [D' | I] -> [I | D'^-1]
  __shared__ double pinv[KLMAX][M2 + 1], pinvi[KLMAX][M2 + 1];  // top kl rows of the previous D'^-1
  __shared__ int s_piv;
  // Interface i reads the spike rows [hi_i - kl, hi_i + kl) (all 2kl columns)
  // and the top rows of partition i, i.e. the lower half of interface i-1's
  // window: a ring of three windows in dynamic shared memory, the next one
  // staged by cp.async while the current interface is factored.
  extern __shared__ __align__(16) double swnd[];  // [3][2 planes][2kl rows][2kl cols]
  const int wsz = 2 * w * w;
  auto stage_win = [&](int ii) {
    if (ii + 1 < a.P) {
      const int h = part_lo(ii + 1, a.n, a.P);
      double* dst = swnd + (size_t)(ii % 3) * wsz;
      for (int e = tid; e < w * w; e += RT) {
        const int rr = e / w, c = e % w;
        const long long o = (long long)(h - kl + rr) * w + c;
        cp_async8(dst + e, Sr + o, true);
        cp_async8(dst + w * w + e, Si + o, true);
      }
    }
    cp_async_commit();
  };
  int cur_i = 0;
  auto sp = [&](int row, int col, double& vr, double& vi) {  // spike buffer entry (windows i-1, i)
    const int h = part_lo(cur_i + 1, a.n, a.P);
    int ii = cur_i, rr = row - (h - kl);
    if (rr < 0) {  // top rows of partition cur_i: lower half of window cur_i - 1
      ii = cur_i - 1;
      rr = row - (part_lo(cur_i, a.n, a.P) - kl);
    }
    const double* src = swnd + (size_t)(ii % 3) * wsz;
    vr = src[rr * w + col];
    vi = src[w * w + rr * w + col];
  };
  stage_win(0);
  for (int i = 0; i + 1 < a.P; ++i) {
    const int hi_i = part_lo(i + 1, a.n, a.P);  // first row of partition i+1
    cur_i = i;
    stage_win(i + 1);
    cp_async_wait<1>();
    __syncthreads();
    // D_i
    for (int e = tid; e < w * w; e += RT) {
      const int r = e / w, c = e % w;
      double vr = (r == c) ? 1.0 : 0.0, vi = 0.0;
      if (r < kl && c >= kl) sp(hi_i - kl + r, c - kl, vr, vi);            // V_i^b
      else if (r >= kl && c < kl) sp(hi_i + (r - kl), kl + c, vr, vi);     // W_{i+1}^t
      ar[r][c] = vr;
      ai[r][c] = vi;
      ar[r][w + c] = (r == c) ? 1.0 : 0.0;
      ai[r][w + c] = 0.0;
    }
    __syncthreads();
    if (i > 0) {
      // F_i (top kl rows) = W_i^b * D'_{i-1}^-1[0:kl, :]
      const int lo_i = part_lo(i, a.n, a.P);
      for (int e = tid; e < kl * w; e += RT) {
        const int r = e / w, c = e % w;
        double s_r = 0.0, s_i = 0.0;
        for (int q = 0; q < kl; ++q) {
          double vr, vi;
          sp(hi_i - kl + r, kl + q, vr, vi);  // W_i^b[r][q]
          s_r += vr * pinv[q][c] - vi * pinvi[q][c];
          s_i += vr * pinvi[q][c] + vi * pinv[q][c];
        }
        Fr[(long long)(i * kl + r) * w + c] = s_r;
        Fi[(long long)(i * kl + r) * w + c] = s_i;
      }
      __syncthreads();
      // D'_i[0:kl, kl:2kl] -= F_i[:, kl:2kl] V_i^t
      for (int e = tid; e < kl * kl; e += RT) {
        const int r = e / kl, c = e % kl;
        double s_r = 0.0, s_i = 0.0;
        for (int q = 0; q < kl; ++q) {
          double vr, vi;
          sp(lo_i + q, c, vr, vi);  // V_i^t[q][c]
          const double f_r = Fr[(long long)(i * kl + r) * w + kl + q];
          const double f_i = Fi[(long long)(i * kl + r) * w + kl + q];
          s_r += f_r * vr - f_i * vi;
          s_i += f_r * vi + f_i * vr;
        }
        ar[r][kl + c] -= s_r;
        ai[r][kl + c] -= s_i;
      }
      __syncthreads();
    }
    // Gauss-Jordan with partial pivoting on [D' | I]
    for (int p = 0; p < w; ++p) {
      if (tid < 32) {
        double best = -1.0;
        int bi = p;
        const int r = p + tid;
        if (r < w) {
          best = hypot(ar[r][p], ai[r][p]);
          bi = r;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
          }
        }
        if (tid == 0) {
          s_piv = bi;
          if (!(best > 0.0)) atomicMin(a.info + k, INT_MAX - 1);
        }
      }
      __syncthreads();
      const int q = s_piv;
      if (q != p)
        for (int c = tid; c < 2 * w; c += RT) {
          double t = ar[p][c];
          ar[p][c] = ar[q][c];
          ar[q][c] = t;
          t = ai[p][c];
          ai[p][c] = ai[q][c];
          ai[q][c] = t;
        }
      __syncthreads();
      const double pr = ar[p][p], pim = ai[p][p];
      const double den = pr * pr + pim * pim;
      const double ir = den > 0.0 ? pr / den : 0.0, ii = den > 0.0 ? -pim / den : 0.0;
      __syncthreads();
      for (int c = tid; c < 2 * w; c += RT) {  // scale row p
        const double x_r = ar[p][c], x_i = ai[p][c];
        ar[p][c] = x_r * ir - x_i * ii;
        ai[p][c] = x_r * ii + x_i * ir;
      }
      __syncthreads();
      for (int e = tid; e < w * 2 * w; e += RT) {  // eliminate column p elsewhere
        const int r = e / (2 * w), c = e % (2 * w);
        if (r == p) continue;
        const double fr2 = ar[r][p], fi2 = ai[r][p];
        if (c == p) continue;
        ar[r][c] -= fr2 * ar[p][c] - fi2 * ai[p][c];
        ai[r][c] -= fr2 * ai[p][c] + fi2 * ar[p][c];
      }
      __syncthreads();
      for (int r = tid; r < w; r += RT)
        if (r != p) {
          ar[r][p] = 0.0;
          ai[r][p] = 0.0;
        }
      __syncthreads();
    }
    for (int e = tid; e < w * w; e += RT) {
      const int r = e / w, c = e % w;
      if (r < kl) {
        pinv[r][c] = ar[r][w + c];
        pinvi[r][c] = ai[r][w + c];
      }
      Dr[(long long)i * w * w + e] = ar[r][w + c];
      Di[(long long)i * w * w + e] = ai[r][w + c];
    }
    __syncthreads();
  }
}

// ---- interface solve: one CTA per (shift, RS_NC-column chunk) ---------------------
// The chain over the P-1 interfaces is sequential; narrow column chunks put
// more CTAs on it (one (row, column) entry per thread) and shorten each step.
constexpr int RS_NC = 8;
struct RSArgs {
  int n, kl, P, nrhs;
  const double *sr, *si;
  long long ss;
  const double *dr, *di, *fr, *fi;
  long long sa;
  const double *xr, *xi;  // g (after the partition solves)
  long long ldx, sx;
  double *yr, *yi;  // interface values [count][P-1][2kl][nrhs]
  long long sy;
};

__global__ void __launch_bounds__(RT) band_rsolve_kernel(RSArgs a) {
  const int k = blockIdx.x, chunk = blockIdx.y, kl = a.kl, w = 2 * kl, tid = threadIdx.x;
  const int c0 = chunk * RS_NC, nc = min(RS_NC, a.nrhs - c0);
  const double* Sr = a.sr + k * a.ss;
  const double* Si = a.si + k * a.ss;
  const double* Dr = a.dr + k * a.sa;
  const double* Di = a.di + k * a.sa;
  const double* Fr = a.fr + k * a.sa;
  const double* Fi = a.fi + k * a.sa;
  const double* Xr = a.xr + k * a.sx;
  const double* Xi = a.xi + k * a.sx;
  double* Yr = a.yr + k * a.sy;
  double* Yi = a.yi + k * a.sy;
  __shared__ double zr[M2][33], zi[M2][33], pr_[M2][33], pi_[M2][33];
  auto yo = [&](int i, int r, int c) { return ((long long)i * w + r) * a.nrhs + c0 + c; };
  // forward: z_i = r_i - F_i z_{i-1} (top kl rows)
  for (int i = 0; i + 1 < a.P; ++i) {
    const int hi_i = part_lo(i + 1, a.n, a.P);
    for (int e = tid; e < w * nc; e += RT) {
      const int r = e / nc, c = e % nc;
      const int row = r < kl ? hi_i - kl + r : hi_i + (r - kl);
      const long long o = (long long)row * a.ldx + c0 + c;
      double vr = Xr[o], vi = Xi[o];
      if (i > 0 && r < kl) {
        for (int q = 0; q < w; ++q) {
          const double f_r = Fr[(long long)(i * kl + r) * w + q], f_i = Fi[(long long)(i * kl + r) * w + q];
          vr -= f_r * pr_[q][c] - f_i * pi_[q][c];
          vi -= f_r * pi_[q][c] + f_i * pr_[q][c];
        }
      }
      zr[r][c] = vr;
      zi[r][c] = vi;
    }
    __syncthreads();
    for (int e = tid; e < w * nc; e += RT) {
      const int r = e / nc, c = e % nc;
      pr_[r][c] = zr[r][c];
      pi_[r][c] = zi[r][c];
      Yr[yo(i, r, c)] = zr[r][c];
      Yi[yo(i, r, c)] = zi[r][c];
    }
    __syncthreads();
  }
  // backward: y_i = D'^-1_i (z_i - (0; V_{i+1}^t y_{i+1}[kl:]))
  for (int i = a.P - 2; i >= 0; --i) {
    const int hi_i = part_lo(i + 1, a.n, a.P);
    for (int e = tid; e < w * nc; e += RT) {
      const int r = e / nc, c = e % nc;
      double vr = Yr[yo(i, r, c)], vi = Yi[yo(i, r, c)];
      if (r >= kl && i + 2 < a.P) {
        for (int q = 0; q < kl; ++q) {  // V_{i+1}^t[r-kl][q] * y_{i+1}[kl+q]
          const long long o = (long long)(hi_i + (r - kl)) * w + q;
          const double v_r = Sr[o], v_i = Si[o];
          vr -= v_r * pr_[kl + q][c] - v_i * pi_[kl + q][c];
          vi -= v_r * pi_[kl + q][c] + v_i * pr_[kl + q][c];
        }
      }
      zr[r][c] = vr;
      zi[r][c] = vi;
    }
    __syncthreads();
    for (int e = tid; e < w * nc; e += RT) {
      const int r = e / nc, c = e % nc;
      double vr = 0.0, vi = 0.0;
      for (int q = 0; q < w; ++q) {
        const double d_r = Dr[(long long)i * w * w + r * w + q], d_i = Di[(long long)i * w * w + r * w + q];
        vr += d_r * zr[q][c] - d_i * zi[q][c];
        vi += d_r * zi[q][c] + d_i * zr[q][c];
      }
      pr_[r][c] = vr;
      pi_[r][c] = vi;
    }
    __syncthreads();
    for (int e = tid; e < w * nc; e += RT) {
      const int r = e / nc, c = e % nc;
      Yr[yo(i, r, c)] = pr_[r][c];
      Yi[yo(i, r, c)] = pi_[r][c];
    }
    __syncthreads();
  }
}

// ---- tips of partition j in spike-column order: T_j = [x_{j+1}^t ; x_{j-1}^b] ----------
// (zero where the neighbour does not exist), so that the correction of every
// partition is one product X_j -= [V_j W_j] T_j.  Item k = blockIdx.y.
struct TGArgs {
  int kl, P, nrhs;
  const double *yr, *yi;
  long long sy;
  double *tr, *ti;
  long long st;
};
__global__ void band_tips_kernel(TGArgs a) {
  const int k = blockIdx.y, w = 2 * a.kl;
  const long long tot = (long long)a.P * w * a.nrhs;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % a.nrhs);
    const long long rq = e / a.nrhs;
    const int q = (int)(rq % w), j = (int)(rq / w);
    double vr = 0.0, vi = 0.0;
    long long o = -1;
    if (q < a.kl) {
      if (j + 1 < a.P) o = ((long long)j * w + a.kl + q) * a.nrhs + c;        // y_j[kl + q]
    } else if (j > 0) {
      o = ((long long)(j - 1) * w + (q - a.kl)) * a.nrhs + c;                  // y_{j-1}[q - kl]
    }
    if (o >= 0) {
      vr = a.yr[k * a.sy + o];
      vi = a.yi[k * a.sy + o];
    }
    a.tr[k * a.st + e] = vr;
    a.ti[k * a.st + e] = vi;
  }
}

// ---- slot-ordered copy of U for the backward sweep (built once per factorization) ----
// The backward sweep keeps each right-hand side's active rows j-2kl..j in
// 2kl+1 registers ("slots") that do not move inside a chunk of SCB rows: at
// the chunk starting with row j1, slot s holds row j1 - s; step jj solves
// slot jj and gives it to the entering row j1 - jj - (2kl+1), so every slot
// index in the unrolled chunk body is a compile-time constant.  Between
// chunks the slots rotate by SCB (register renaming at the loop edge, paid
// once per chunk).  The U column of step j is re-ordered to match, once:
// Us[j][s] = U(row in slot s, j), 0 for row j's own slot,
// Us[j][2kl+1] = 1 / U(j, j).
__host__ __device__ constexpr int bwd_chunk(int kl) { return 2 * kl + 1 < 8 ? 2 * kl + 1 : 8; }

struct SOArgs {
  int n, kl, P;
  const double *wr, *wi;
  long long sw;
  double2* us;  // item 0; item k at + k*sa doubles
  long long sa;
};

__global__ void band_slot_bwd_kernel(SOArgs a) {
  const int k = blockIdx.y, kl = a.kl, KV = 2 * kl, NB = KV + 1, LW = 3 * kl + 1, NU = NB + 1;
  const double* Wr = a.wr + k * a.sw;
  const double* Wi = a.wi + k * a.sw;
  double2* Us = reinterpret_cast<double2*>(reinterpret_cast<double*>(a.us) + k * a.sa);
  const long long total = (long long)a.n * NU;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / NU), s = (int)(e % NU);
    int part = (int)(((long long)j * a.P) / a.n);
    while (part + 1 < a.P && part_lo(part + 1, a.n, a.P) <= j) ++part;
    while (part_lo(part, a.n, a.P) > j) --part;
    const int top = part_lo(part + 1, a.n, a.P) - 1, head = (top - j) % bwd_chunk(kl);
    double2 v = make_double2(0.0, 0.0);
    if (s == NB) {
      const double dr = Wr[(long long)j * LW + KV], di = Wi[(long long)j * LW + KV];
      const double den = dr * dr + di * di;
      if (den > 0.0) v = make_double2(dr / den, -di / den);
    } else if (s != head) {
      // step head of its chunk: row j - d (d = 1..KV) sits in slot (head + d) mod NB, U entry KV - d
      int d = s - head;
      if (d < 0) d += NB;
      v = make_double2(Wr[(long long)j * LW + KV - d], Wi[(long long)j * LW + KV - d]);
    }
    Us[e] = v;
  }
}

// ---- staged partition solves: one CTA per (partition, shift, column block) -------
// One thread per right-hand side keeps its column's active rows in registers;
// all threads of a CTA share the factor columns, staged through shared memory
// in chunks of rows by cp.async (double buffered, re/im interleaved so one
// LDS.128 feeds a complex multiply-add) together with the right-hand-side rows
// that will ENTER the window during the chunk.  The shift index is the fastest
// grid index, so the CTAs that read the same rows of a shared right-hand side
// run together (L2).  Forward (pivots + unit L) and backward (U) are separate
// kernels so each keeps its own register window.
constexpr int SNW = 3;   // warps per CTA (96 right-hand sides)
constexpr int SC = 8;    // forward sweep rows per staged chunk
constexpr int NST = 3;   // staged chunks in flight (the loads of a chunk are issued NST-1 chunks ahead)
size_t sweep_xring_bytes(int nt, int sc) { return sizeof(double) * NST * sc * 2 * (size_t)nt; }

// One forward step with the row interchange (0 <-> P) folded in at compile
// time: x0 = w[P]; the window slides by one as each multiply-add writes row
// i+1's update into slot i.  The caller dispatches on the warp-uniform P with
// a switch (17 straight-line bodies; measured faster than an in-place swap
// followed by one shared body, whose register renaming costs more moves).
template <int KL, int P>
__device__ __forceinline__ void fwd_step(double (&wr)[KL + 1], double (&wi)[KL + 1], const double2* __restrict__ l,
                                         double& x0r, double& x0i) {
  x0r = wr[P];
  x0i = wi[P];
  const double o_r = wr[0], o_i = wi[0];
#pragma unroll
  for (int i = 0; i < KL; ++i) {
    const double sr = (i + 1 == P) ? o_r : wr[i + 1];
    const double si = (i + 1 == P) ? o_i : wi[i + 1];
    const double2 lv = l[i];
    wr[i] = fma(-lv.x, x0r, fma(lv.y, x0i, sr));
    wi[i] = fma(-lv.x, x0i, fma(-lv.y, x0r, si));
  }
}

template <int KL>
__global__ void __launch_bounds__(SNW * 32, 4) band_psolve_fwd_kernel(PSArgs a) {
  constexpr int KV = 2 * KL, LW = 3 * KL + 1;
  const int k = blockIdx.x % a.count, part = blockIdx.x / a.count, tid = threadIdx.x, nt = blockDim.x;
  const int col = blockIdx.y * nt + tid;
  const bool on = col < a.nrhs;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const double* Wr = a.wr + k * a.sw;
  const double* Wi = a.wi + k * a.sw;
  const int* ipiv = a.ipiv + k * a.sp;
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  const bool sep = a.fr != nullptr;
  const double* Fr = sep ? a.fr + k * a.sf : Xr;
  const double* Fi = sep ? (a.fi ? a.fi + k * a.sf : nullptr) : Xi;
  const long long ldf = sep ? a.ldf : a.ldx;
  extern __shared__ __align__(16) double sx[];  // [NST buf][SC rows][nt] (re, im)
  __shared__ double2 sl[NST][SC][KL];           // multipliers (re, im) of column j
  __shared__ int spv[NST][SC];
  const int xbase = lo + KL + 1;  // row entering the window at step lo
  auto stage = [&](int buf, int c) {
    const int j0 = lo + c * SC;
    for (int e = tid; e < SC * KL; e += nt) {
      const int jj = e / KL, i = e % KL, j = j0 + jj;
      const bool ok = j < hi;
      const long long o = ok ? (long long)j * LW + KV + 1 + i : 0;
      cp_async8(&sl[buf][jj][i].x, Wr + o, ok);
      cp_async8(&sl[buf][jj][i].y, Wi + o, ok);
    }
    for (int jj = tid; jj < SC; jj += nt) cp_async4(&spv[buf][jj], ipiv + min(j0 + jj, hi - 1), j0 + jj < hi);
    double* xb = sx + (size_t)buf * SC * 2 * nt + 2 * tid;
    const double* fr = Fr + (long long)(xbase + c * SC) * ldf + col;
    const double* fi = Fi ? Fi + (long long)(xbase + c * SC) * ldf + col : nullptr;
#pragma unroll
    for (int r = 0; r < SC; ++r) {
      const bool ok = on && xbase + c * SC + r < hi;
      cp_async8(xb + r * 2 * nt, ok ? fr + r * ldf : Fr, ok);
      cp_async8(xb + r * 2 * nt + 1, ok && fi ? fi + r * ldf : Fr, ok && fi != nullptr);
    }
    cp_async_commit();
  };
  double wr_[KL + 1], wi_[KL + 1];
#pragma unroll
  for (int i = 0; i <= KL; ++i) {
    wr_[i] = wi_[i] = 0.0;
    if (on && lo + i < hi) {
      const long long o = (long long)(lo + i) * ldf + col;
      wr_[i] = Fr[o];
      if (Fi) wi_[i] = Fi[o];
    }
  }
  double* pxr = Xr + (long long)lo * a.ldx + col;
  double* pxi = Xi + (long long)lo * a.ldx + col;
  const int nch = (hi - lo + SC - 1) / SC;
#pragma unroll
  for (int c = 0; c < NST - 1; ++c) stage(c, c);  // chunks past the end: all zero-filled
  int buf = 0;
  for (int c = 0; c < nch; ++c) {
    stage(buf == 0 ? NST - 1 : buf - 1, c + NST - 1);
    cp_async_wait<NST - 1>();
    __syncthreads();
    const int j0 = lo + c * SC, jn = min(SC, hi - j0);
    const double2* xb = reinterpret_cast<const double2*>(sx + (size_t)buf * SC * 2 * nt) + tid;
#pragma unroll 1
    for (int jj = 0; jj < jn; ++jj) {
      const int p = spv[buf][jj] - (j0 + jj);
      const double2* lcol = sl[buf][jj];
      double x0r, x0i;
#define FB_FWD_CASE(I)                                                          \
  case I:                                                                       \
    if constexpr (I <= KL) fwd_step<KL, (I <= KL ? I : 0)>(wr_, wi_, lcol, x0r, x0i); \
    break;
      switch (p) {
        FB_FWD_CASE(1) FB_FWD_CASE(2) FB_FWD_CASE(3) FB_FWD_CASE(4) FB_FWD_CASE(5) FB_FWD_CASE(6)
        FB_FWD_CASE(7) FB_FWD_CASE(8) FB_FWD_CASE(9) FB_FWD_CASE(10) FB_FWD_CASE(11) FB_FWD_CASE(12)
        FB_FWD_CASE(13) FB_FWD_CASE(14) FB_FWD_CASE(15) FB_FWD_CASE(16)
        default: fwd_step<KL, 0>(wr_, wi_, lcol, x0r, x0i); break;
      }
#undef FB_FWD_CASE
      if (on) {
        *pxr = x0r;
        *pxi = x0i;
      }
      pxr += a.ldx;
      pxi += a.ldx;
      const double2 nv = xb[jj * nt];
      wr_[KL] = nv.x;
      wi_[KL] = nv.y;
    }
    buf = buf + 1 == NST ? 0 : buf + 1;
    __syncthreads();
  }
  cp_async_wait<0>();
}

// Backward sweep (slots as described above the re-ordering kernel): step jj
// of a chunk solves slot jj, x = w[jj] / U_jj, the entering row takes slot jj,
// and every slot is updated with its U entry (0 for slot jj) by straight-line
// multiply-adds on fixed registers.  Staging: the chunk's U columns are one
// contiguous run of the slot-ordered copy and every entering right-hand-side
// row is one contiguous run per plane, so ONE elected thread moves a chunk with
// 1 + 2*SCB bulk copies (cp.async.bulk, the TMA engine) that complete on the
// chunk's mbarrier -- the other threads carry no staging code or registers.
// Rows past the partition start are not copied: their U entries are zero, so
// whatever sits in the ring never reaches a stored value.
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, void* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Each right-hand side is carried by TWO adjacent lanes: the even lane holds the
// real parts of the 2KL+1 active rows, the odd lane the imaginary parts (half
// the registers per thread, twice the warps per SM).  Both lanes run the same
// code: w -= u.x*q1 - u.y*q2 with (q1, q2) = (q_re, q_im) for the real lane and
// (q_im, -q_re) for the imaginary lane; the solved value's other component
// comes from the partner lane by one shuffle.
// BULK = false (odd leading dimension: rows not 16-byte aligned): every thread
// stages its own entries with cp.async instead, same ring layout.
constexpr int BNC = 48;  // right-hand sides per CTA of the backward sweep (96 threads: 5 CTAs per SM at 128 registers)

template <int KL, bool BULK>
__global__ void __launch_bounds__(2 * BNC, 5) band_psolve_bwd_kernel(PSArgs a) {
  constexpr int KV = 2 * KL, NB = KV + 1, NU = NB + 1, SCB = bwd_chunk(KL);
  const int k = blockIdx.x % a.count, part = blockIdx.x / a.count, tid = threadIdx.x;
  const int nc = blockDim.x >> 1;  // columns of this CTA
  const int col0 = blockIdx.y * nc, col = col0 + (tid >> 1);
  const bool im = tid & 1;
  const bool on = col < a.nrhs;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const double2* Us = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(a.us) + k * a.sa);
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  double* Xo = im ? Xi : Xr;  // this lane's plane
  extern __shared__ __align__(16) double sx[];  // [NST buf][2 planes][SCB rows][nc]
  __shared__ __align__(16) double2 su[NST][SCB * NU];
  __shared__ __align__(8) unsigned long long full[NST];
  const int top = hi - 1;
  // columns of this CTA, rounded up to a whole 16 bytes (the pad column exists: ldx is even)
  const unsigned rowbytes = 8u * (unsigned)((min(nc, a.nrhs - col0) + 1) & ~1);
  if (BULK && tid == 0) {
#pragma unroll
    for (int b = 0; b < NST; ++b) mbar_init(&full[b], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto stage = [&](int buf, int c) {
    const int j1 = top - c * SCB, jl = max(j1 - SCB + 1, lo);
    const int r0 = j1 - NB;                       // row entering at step j1; step j1 - r takes row r0 - r
    const int nr = max(0, min(SCB, r0 - lo + 1));  // rows r0, r0-1, ... that exist
    double* xb = sx + (size_t)buf * 2 * SCB * nc;
    if constexpr (BULK) {  // elected thread only
      unsigned bytes = 0;
      if (jl <= j1) bytes = (unsigned)(j1 - jl + 1) * NU * 16u;
      // the buffer was read through the generic proxy (the __syncthreads that freed it orders
      // those reads before this thread); the bulk copies write it through the async proxy
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive_expect_tx(&full[buf], bytes + 2u * nr * rowbytes);
      if (bytes) bulk_g2s(&su[buf][(size_t)(jl - (j1 - SCB + 1)) * NU], Us + (long long)jl * NU, bytes, &full[buf]);
      const double* fr = Xr + (long long)r0 * a.ldx + col0;
      const double* fi = Xi + (long long)r0 * a.ldx + col0;
#pragma unroll 1
      for (int r = 0; r < nr; ++r) {
        bulk_g2s(xb + r * nc, fr - r * a.ldx, rowbytes, &full[buf]);
        bulk_g2s(xb + (SCB + r) * nc, fi - r * a.ldx, rowbytes, &full[buf]);
      }
    } else {
      const int jb = j1 - SCB + 1;
      for (int e = tid; e < SCB * NU; e += blockDim.x) {
        const bool ok = jb + e / NU >= lo;
        cp_async16(&su[buf][e], ok ? Us + (long long)jb * NU + e : Us, ok ? 16 : 0);
      }
#pragma unroll 1
      for (int r = 0; r < SCB; ++r) {
        const bool ok = on && r < nr;
        cp_async8(xb + ((im ? SCB : 0) + r) * nc + (tid >> 1), ok ? Xo + (long long)(r0 - r) * a.ldx + col : Xo, ok);
      }
      cp_async_commit();
    }
  };
  double w_[NB];  // slot s = this lane's component of row j1 - s of the current chunk
#pragma unroll
  for (int s = 0; s < NB; ++s) w_[s] = (on && top - s >= lo) ? Xo[(long long)(top - s) * a.ldx + col] : 0.0;
  double* px = Xo + (long long)top * a.ldx + col;
  const int nch = (hi - lo + SCB - 1) / SCB;
  if (!BULK || tid == 0) {
#pragma unroll 1
    for (int c = 0; c < NST - 1; ++c) stage(c, c);
  }
  int buf = 0;
  unsigned phase = 0;
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    // the buffer staged now was released at the end of chunk c-1
    if (!BULK || tid == 0) stage(buf == 0 ? NST - 1 : buf - 1, c + NST - 1);
    if constexpr (BULK) {
      mbar_wait_parity(&full[buf], phase);
    } else {
      cp_async_wait<NST - 1>();
      __syncthreads();
    }
    const int j1 = top - c * SCB;
    const double* xb = sx + (size_t)buf * 2 * SCB * nc + (im ? SCB * nc : 0) + (tid >> 1);
#pragma unroll
    for (int jj = 0; jj < SCB; ++jj) {
      const double nv = xb[jj * nc];
      const double2* ucol = &su[buf][(SCB - 1 - jj) * NU];
      const double2 dv = ucol[NB];
      const double yo = w_[jj];
      w_[jj] = nv;
      const double yp = __shfl_xor_sync(0xffffffffu, yo, 1);  // the partner lane's component
      const double yr = im ? yp : yo, yi = im ? yo : yp;
      const double qr = yr * dv.x - yi * dv.y, qi = yr * dv.y + yi * dv.x;
      const double q1 = im ? qi : qr, q2 = im ? -qr : qi;
#pragma unroll
      for (int s = 0; s < NB; ++s) {  // slot jj (the entering row) has U entry 0
        if (s % 8 == 7) asm volatile("" ::: "memory");  // keep the loads of u in groups of 8 (registers)
        const double2 uv = ucol[s];
        w_[s] = fma(-uv.x, q1, fma(uv.y, q2, w_[s]));
      }
      if (on && j1 - jj >= lo) px[-(long long)jj * a.ldx] = q1;
    }
    px -= (long long)SCB * a.ldx;
    {  // rotate the slots by SCB for the next chunk
      double t[NB];
#pragma unroll
      for (int s = 0; s < NB; ++s) t[s] = w_[(s + SCB) % NB];
#pragma unroll
      for (int s = 0; s < NB; ++s) w_[s] = t[s];
    }
    if (++buf == NST) {
      buf = 0;
      phase ^= 1;
    }
    __syncthreads();  // every thread is done with the chunk's buffer
  }
  if constexpr (!BULK) cp_async_wait<0>();
}

// ---- backward sweep on the FP64 tensor pipe (kl = 16) -----------------------------
// The SIMT sweeps above feed every complex multiply-add (4 DFMA) with one
// 16-byte broadcast shared-memory load; the register-file fill of those loads
// (512 B per warp and load), not the FP64 pipe, bounds them (~40 % of the pipe,
// profiles/).  Here the sweep runs in steps of FOUR rows: the 4 x 4 diagonal
// block is solved by substitution (SIMT, two quad shuffles), and the rank-4
// update of the 32 rows above is a DMMA product W^T(8 columns x 8 rows) +=
// X^T(8 x 4) * (-U^T)(4 x 8) per row tile, whose B fragments are read as one
// distinct double per lane (256 B per warp and 256 multiply-adds): 7 x less
// operand traffic per flop.  A warp owns 8 right-hand sides; the active rows
// (36, plus the 4 entering next) live in 40 fixed accumulator slots, slot =
// (distance from the partition's last row) mod 40, so the 10 steps of one turn
// of the slots are unrolled with compile-time tile indices.  The factor is
// re-ordered once per factorization into exactly this fragment order (T4).
constexpr int T4_NT = 5, T4_SLOTS = 40, T4_PERIOD = 10;
constexpr int T4_STEPD = T4_NT * 2 * 32 + 32;  // doubles per 4-row step: B fragments + the 4x4 block (re, im)
constexpr int T4_S = 2;                        // steps per staged chunk
constexpr int T4_WARPS = 4;                    // 32 right-hand sides per CTA
constexpr int T4_NST = 5;                      // staged chunks in flight (9.7 KB each)
constexpr int T4_CHUNKD = T4_S * T4_STEPD + 2 * 4 * T4_S * 8 * T4_WARPS;  // + entering rows [plane][row][32 columns]

__host__ __device__ inline long long t4_steps(int n, int P) { return (part_sz(n, P) + 3) / 4; }

struct T4Args {
  int n, P;
  const double *wr, *wi;
  long long sw;
  double* t4;  // item 0; item k at + k*sa doubles
  long long sa;
};

__global__ void band_t4_kernel(T4Args a) {
  constexpr int KV = 32, LW = 49;
  const int k = blockIdx.y;
  const double* Wp[2] = {a.wr + k * a.sw, a.wi + k * a.sw};
  double* T = a.t4 + k * a.sa;
  const long long spp = t4_steps(a.n, a.P), total = spp * a.P * T4_STEPD;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long gs = e / T4_STEPD;
    const int r = (int)(e % T4_STEPD), part = (int)(gs / spp), s = (int)(gs % spp);
    const int lo = part_lo(part, a.n, a.P), top = part_lo(part + 1, a.n, a.P) - 1;
    double v = 0.0;
    if (r < T4_NT * 64) {
      const int t = r >> 6, plane = (r >> 5) & 1, l = r & 31, kk = l & 3, nn = l >> 2;
      const int slot = 8 * t + nn;
      const int delta = ((slot - 4 * s) % T4_SLOTS + T4_SLOTS) % T4_SLOTS;  // row = top - (4s + delta)
      const int d = delta - kk;                                             // rows above the solved row kk
      const int rcol = top - (4 * s + kk), rrow = rcol - d;
      if (delta >= 4 && delta < 36 && d >= 1 && d <= KV && rrow >= lo) v = -Wp[plane][(long long)rcol * LW + KV - d];
    } else {
      const int idx = r - T4_NT * 64, c = idx >> 1, plane = idx & 1, kk = c >> 2, kp = c & 3;
      const int rk = top - (4 * s + kk), rp = top - (4 * s + kp);
      if (rk >= lo) {
        if (kp == kk) {
          const double dr = Wp[0][(long long)rk * LW + KV], di = Wp[1][(long long)rk * LW + KV];
          const double den = dr * dr + di * di;
          if (den > 0.0) v = plane ? -di / den : dr / den;
        } else if (kp < kk) {
          v = Wp[plane][(long long)rp * LW + KV - (kk - kp)];  // U(row rk, column rp)
        }
      }
    }
    T[e] = v;
  }
}

__global__ void __launch_bounds__(T4_WARPS * 32, 4) band_psolve_bwd_t4_kernel(PSArgs a) {
  // column group fastest, then shift: the CTAs that read the same T4 run together (L2)
  const int ncg = (a.nrhs + 8 * T4_WARPS - 1) / (8 * T4_WARPS);
  const int cgi = blockIdx.x % ncg, k = (blockIdx.x / ncg) % a.count, part = blockIdx.x / (ncg * a.count);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int col0 = cgi * 8 * T4_WARPS, col = col0 + warp * 8 + g;
  const bool on = col < a.nrhs;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P), top = hi - 1;
  const long long spp = t4_steps(a.n, a.P);
  const double* T4 = a.t4 + k * a.sa + (long long)part * spp * T4_STEPD;
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  extern __shared__ __align__(16) double sx[];  // [T4_NST][T4_CHUNKD]
  __shared__ __align__(8) unsigned long long full[T4_NST];
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < T4_NST; ++b) mbar_init(&full[b], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int nsteps = (hi - lo + 3) / 4, nchunks = (nsteps + T4_S - 1) / T4_S;
  // Staging of chunk c (steps c*T4_S ..): the factor fragments are one contiguous
  // run -> one bulk copy (TMA engine) by an elected thread onto the chunk's
  // mbarrier; the 4*T4_S entering right-hand-side rows (32 columns, 2 planes) are
  // spread over the CTA as 8-byte cp.async (zero-filled where the row or column
  // does not exist), one commit group per chunk.
  constexpr int XE = 2 * 4 * T4_S * 8 * T4_WARPS;  // entering-row entries per chunk
  auto stage = [&](int buf, int c) {
    double* dst = sx + (size_t)buf * T4_CHUNKD;
    const int s0 = c * T4_S;
    if (tid == 0) {
      const unsigned bytes = c < nchunks ? (unsigned)(T4_S * T4_STEPD * 8) : 0u;
      // generic-proxy reads of the freed buffer (ordered before this thread by the
      // __syncthreads that freed it) -> async-proxy refill
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive_expect_tx(&full[buf], bytes);
      if (bytes) bulk_g2s(dst, T4 + (long long)s0 * T4_STEPD, bytes, &full[buf]);
    }
    double* xb = dst + T4_S * T4_STEPD;
    const int rfirst = top - (4 * s0 + T4_SLOTS);  // entering rows of step s: top - (4s + 40 + kk)
#pragma unroll
    for (int e = tid; e < XE; e += T4_WARPS * 32) {
      const int cc_ = e % (8 * T4_WARPS), rr = (e / (8 * T4_WARPS)) % (4 * T4_S), pl = e / (8 * T4_WARPS * 4 * T4_S);
      const int r = rfirst - rr;
      const bool ok = c < nchunks && r >= lo && col0 + cc_ < a.nrhs;
      const double* src = (pl ? Xi : Xr) + (ok ? (long long)r * a.ldx + col0 + cc_ : 0);
      cp_async8(xb + e, src, ok);
    }
    cp_async_commit();
  };
  // accumulator slots: tile t, lane (g, q) holds slots 8t + 2q + {0, 1} of column g
  double cr[T4_NT][2], ci[T4_NT][2];
#pragma unroll
  for (int t = 0; t < T4_NT; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = top - (8 * t + 2 * q + e);
      cr[t][e] = ci[t][e] = 0.0;
      if (on && r >= lo) {
        cr[t][e] = Xr[(long long)r * a.ldx + col];
        ci[t][e] = Xi[(long long)r * a.ldx + col];
      }
    }
#pragma unroll 1
  for (int c = 0; c < T4_NST - 1; ++c) stage(c, c);
  int buf = 0;
  unsigned phase = 0;
  const int quad = lane & ~3;
  constexpr int CPT = T4_PERIOD / T4_S;  // chunks per turn of the slots
#pragma unroll 1
  for (int c0 = 0; c0 < nchunks; c0 += CPT) {
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      const int c = c0 + cc;  // chunks past nchunks: nothing staged, nothing stored
      cp_async_wait<T4_NST - 2>();          // this thread's entering-row copies of chunk c
      mbar_wait_parity(&full[buf], phase);  // the chunk's factor fragments
      __syncthreads();                      // all copies of chunk c visible; chunk c-1's buffer is free
      stage(buf == 0 ? T4_NST - 1 : buf - 1, c + T4_NST - 1);
      const double* base = sx + (size_t)buf * T4_CHUNKD;
#pragma unroll
      for (int jj = 0; jj < T4_S; ++jj) {
        const int u = cc * T4_S + jj;            // compile-time position in the turn
        const int tu = (4 * u) / 8, h = u & 1;   // solved slots 4u..4u+3: tile tu, lanes q = 2h, 2h+1
        const int s = c * T4_S + jj;
        const double* sd = base + jj * T4_STEPD;
        const double2* D = reinterpret_cast<const double2*>(sd + T4_NT * 64);  // [kk][kp]
        // -- the 4 x 4 block by substitution: lane 2h holds rows 0, 1, lane 2h+1 rows 2, 3
        const double w0r = cr[tu][0], w0i = ci[tu][0], w1r = cr[tu][1], w1i = ci[tu][1];
        auto cmul = [](double ar, double ai, double2 b, double& orr, double& oi) {
          orr = ar * b.x - ai * b.y;
          oi = ar * b.y + ai * b.x;
        };
        double x0r, x0i, x1r, x1i, x2r, x2i, x3r, x3i, tr_, ti_;
        cmul(w0r, w0i, D[0], x0r, x0i);
        {
          const double2 u10 = D[4];
          tr_ = fma(-u10.x, x0r, fma(u10.y, x0i, w1r));
          ti_ = fma(-u10.x, x0i, fma(-u10.y, x0r, w1i));
          cmul(tr_, ti_, D[5], x1r, x1i);
        }
        const int srcA = quad | (2 * h);
        x0r = __shfl_sync(0xffffffffu, x0r, srcA); x0i = __shfl_sync(0xffffffffu, x0i, srcA);
        x1r = __shfl_sync(0xffffffffu, x1r, srcA); x1i = __shfl_sync(0xffffffffu, x1i, srcA);
        {
          const double2 u20 = D[8], u21 = D[9];
          tr_ = fma(-u20.x, x0r, fma(u20.y, x0i, w0r));
          ti_ = fma(-u20.x, x0i, fma(-u20.y, x0r, w0i));
          tr_ = fma(-u21.x, x1r, fma(u21.y, x1i, tr_));
          ti_ = fma(-u21.x, x1i, fma(-u21.y, x1r, ti_));
          cmul(tr_, ti_, D[10], x2r, x2i);
          const double2 u30 = D[12], u31 = D[13], u32 = D[14];
          tr_ = fma(-u30.x, x0r, fma(u30.y, x0i, w1r));
          ti_ = fma(-u30.x, x0i, fma(-u30.y, x0r, w1i));
          tr_ = fma(-u31.x, x1r, fma(u31.y, x1i, tr_));
          ti_ = fma(-u31.x, x1i, fma(-u31.y, x1r, ti_));
          tr_ = fma(-u32.x, x2r, fma(u32.y, x2i, tr_));
          ti_ = fma(-u32.x, x2i, fma(-u32.y, x2r, ti_));
          cmul(tr_, ti_, D[15], x3r, x3i);
        }
        const int srcB = quad | (2 * h + 1);
        x2r = __shfl_sync(0xffffffffu, x2r, srcB); x2i = __shfl_sync(0xffffffffu, x2i, srcB);
        x3r = __shfl_sync(0xffffffffu, x3r, srcB); x3i = __shfl_sync(0xffffffffu, x3i, srcB);
        // A fragment: lane (g, q) carries x_q of column g; the same lane stores it
        const double ar = q == 0 ? x0r : (q == 1 ? x1r : (q == 2 ? x2r : x3r));
        const double ai = q == 0 ? x0i : (q == 1 ? x1i : (q == 2 ? x2i : x3i));
        const int rs = top - (4 * s + q);
        if (on && rs >= lo) {
          Xr[(long long)rs * a.ldx + col] = ar;
          Xi[(long long)rs * a.ldx + col] = ai;
        }
        // the rows entering take the solved slots (first needed two steps on)
        if ((q >> 1) == h) {
          const double* xb = base + T4_S * T4_STEPD + (jj * 4 + 2 * (q & 1)) * 8 * T4_WARPS + warp * 8 + g;
          cr[tu][0] = xb[0];
          cr[tu][1] = xb[8 * T4_WARPS];
          ci[tu][0] = xb[4 * T4_S * 8 * T4_WARPS];
          ci[tu][1] = xb[(4 * T4_S + 1) * 8 * T4_WARPS];
        }
        // -- rank-4 update of every slot (B = -U^T in fragment order; 0 for the solved slots)
        const double nai = -ai;
#pragma unroll
        for (int t = 0; t < T4_NT; ++t) {
          const double br = sd[(t * 2) * 32 + lane], bi = sd[(t * 2 + 1) * 32 + lane];
          dmma(cr[t][0], cr[t][1], ar, br);
          dmma(cr[t][0], cr[t][1], nai, bi);
          dmma(ci[t][0], ci[t][1], ar, bi);
          dmma(ci[t][0], ci[t][1], ai, br);
        }
      }
      if (++buf == T4_NST) {
        buf = 0;
        phase ^= 1;
      }
    }
  }
  cp_async_wait<0>();
}

// ---- fused spike correction + quadrature accumulation ---------------------------
// Q -= sum_t coeff_t * (g_t - [V W]_t T_t): the correction product runs on the
// FP64 tensor pipe with the accumulators starting from the partition solve g
// (read once, never rewritten) and the quadrature term of every shift is folded
// into Q held in registers (kernel.py:108-124 arithmetic, term by term in the
// caller's order), so one contour pass reads each g and spike row once and
// writes Q once.  One CTA = (partition, FA_CHUNK-row chunk, 48-column group);
// a warp owns 8-row tiles.  The K index of the product is permuted (lane
// quarter q owns k = q*KS .. q*KS+KS-1) so that every lane reads its spike
// entries as one contiguous run; the (negated) tips are staged in shared
// memory in B-fragment order under the same permutation.
constexpr int FA_NT = 6;        // 8-column DMMA tiles per warp
constexpr int FA_COLS = FA_NT * 8;
constexpr int FA_CHUNK = 1024;  // rows per CTA
constexpr int FA_MAXG = 8;      // terms whose tips are staged together (24 KB each at kl = 16)
constexpr int FA_KS = 2 * KLMAX / 4;

struct FAArgs {
  int n, kl, P, nrhs, nterms, chunks;
  const double *sr, *si;
  long long ss;
  const double *tr, *ti;  // tips [item][P][2kl][nrhs]
  long long st;
  const double *xr, *xi;  // partition solves g [item][n][ldx]
  long long ldx, sx;
  double *qr, *qi;
  long long ldq;
  int item[kMaxAccTerms], mode[kMaxAccTerms];
  double h[kMaxAccTerms], cr[kMaxAccTerms], ci[kMaxAccTerms];
};

__device__ __forceinline__ double dneg_(double v) {
  return __longlong_as_double(__double_as_longlong(v) ^ 0x8000000000000000ull);
}

template <bool CQ, int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, 1) band_correct_accumulate_kernel(const __grid_constant__ FAArgs a) {
  extern __shared__ double sT[];  // [G][2 planes][KS][FA_NT][32 lanes] = -tips in B-fragment order
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NTHREADS / 32;
  const int g = lane >> 2, q = lane & 3;
  const int part = blockIdx.x / a.chunks, chunk = blockIdx.x % a.chunks;
  const int c0 = blockIdx.y * FA_COLS;
  const int w = 2 * a.kl, KS = (w + 3) / 4;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const int r_begin = lo + chunk * FA_CHUNK, r_end = min(hi, r_begin + FA_CHUNK);
  if (r_begin >= r_end) return;
  const bool vx = (a.ldx & 1) == 0 && (a.sx & 1) == 0;  // 16-byte g loads
  const bool vs = (KS & 1) == 0;                         // 16-byte spike loads
  const int plane = KS * FA_NT * 32;
  for (int t0 = 0; t0 < a.nterms; t0 += FA_MAXG) {
    const int G = min(FA_MAXG, a.nterms - t0);
    __syncthreads();
    for (int e = tid; e < G * 2 * plane; e += NTHREADS) {
      const int l = e & 31;
      int rest = e >> 5;
      const int t = rest % FA_NT;
      rest /= FA_NT;
      const int j = rest % KS;
      rest /= KS;
      const int pl = rest & 1, ti = rest >> 1;
      const int k = (l & 3) * KS + j, col = c0 + t * 8 + (l >> 2);
      double v = 0.0;
      if (k < w && col < a.nrhs) {
        const double* src = (pl ? a.ti : a.tr) + a.item[t0 + ti] * a.st;
        v = -src[((long long)part * w + k) * a.nrhs + col];
      }
      sT[e] = v;
    }
    __syncthreads();
    for (int r0 = r_begin + warp * 8; r0 < r_end; r0 += NW * 8) {
      const int row = r0 + g;
      const bool rok = row < r_end;
      double q_r[FA_NT][2], q_i[FA_NT][2];
#pragma unroll
      for (int t = 0; t < FA_NT; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = c0 + t * 8 + 2 * q + e;
          const bool ok = rok && col < a.nrhs;
          q_r[t][e] = ok ? a.qr[(long long)row * a.ldq + col] : 0.0;
          q_i[t][e] = (CQ && ok) ? a.qi[(long long)row * a.ldq + col] : 0.0;
        }
      for (int ti = 0; ti < G; ++ti) {
        const int it = a.item[t0 + ti];
        const double* Sr = a.sr + it * a.ss + (long long)row * w + q * KS;
        const double* Si = a.si + it * a.ss + (long long)row * w + q * KS;
        const double* Xr = a.xr + it * a.sx + (long long)row * a.ldx;
        const double* Xi = a.xi + it * a.sx + (long long)row * a.ldx;
        double s_r[FA_KS], s_i[FA_KS], c_r[FA_NT][2], c_i[FA_NT][2];
        if (vs) {
#pragma unroll
          for (int j = 0; j < FA_KS; j += 2) {
            double2 vr = make_double2(0.0, 0.0), vi = vr;
            if (rok && j < KS && q * KS + j < w) {
              vr = __ldcs(reinterpret_cast<const double2*>(Sr + j));
              vi = __ldcs(reinterpret_cast<const double2*>(Si + j));
            }
            s_r[j] = vr.x; s_r[j + 1] = vr.y;
            s_i[j] = vi.x; s_i[j + 1] = vi.y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < FA_KS; ++j) {
            const bool ok = rok && j < KS && q * KS + j < w;
            s_r[j] = ok ? __ldcs(Sr + j) : 0.0;
            s_i[j] = ok ? __ldcs(Si + j) : 0.0;
          }
        }
        // the correction product is accumulated from zero and subtracted from g
        // ONCE (accumulating onto g would round every one of the 2kl multiply-adds
        // at |g|'s magnitude, tools/dmma_rounding.py); the loads of g are issued
        // before the products so their latency hides behind the DMMAs
        double g_r[FA_NT][2], g_i[FA_NT][2];
#pragma unroll
        for (int t = 0; t < FA_NT; ++t) {
          const int col = c0 + t * 8 + 2 * q;
          if (vx && rok && col + 1 < a.nrhs) {
            const double2 vr = __ldcs(reinterpret_cast<const double2*>(Xr + col));
            const double2 vi = __ldcs(reinterpret_cast<const double2*>(Xi + col));
            g_r[t][0] = vr.x; g_r[t][1] = vr.y;
            g_i[t][0] = vi.x; g_i[t][1] = vi.y;
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool ok = rok && col + e < a.nrhs;
              g_r[t][e] = ok ? __ldcs(Xr + col + e) : 0.0;
              g_i[t][e] = ok ? __ldcs(Xi + col + e) : 0.0;
            }
          }
        }
#pragma unroll
        for (int t = 0; t < FA_NT; ++t) c_r[t][0] = c_r[t][1] = c_i[t][0] = c_i[t][1] = 0.0;
        const double* br_ = sT + (size_t)(ti * 2) * plane + lane;
        const double* bi_ = br_ + plane;
#pragma unroll
        for (int j = 0; j < FA_KS; ++j) {
          if (j < KS) {
            const double ar = s_r[j], ai = s_i[j], nai = dneg_(ai);
#pragma unroll
            for (int t = 0; t < FA_NT; ++t) {
              const double tr_ = br_[(j * FA_NT + t) * 32], ti_ = bi_[(j * FA_NT + t) * 32];  // -T
              dmma(c_r[t][0], c_r[t][1], ar, tr_);    // - S_r T_r
              dmma(c_r[t][0], c_r[t][1], nai, ti_);   // + S_i T_i
              dmma(c_i[t][0], c_i[t][1], ar, ti_);    // - S_r T_i
              dmma(c_i[t][0], c_i[t][1], ai, tr_);    // - S_i T_r
            }
          }
        }
#pragma unroll
        for (int t = 0; t < FA_NT; ++t)  // x = g + (-S T)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            c_r[t][e] += g_r[t][e];
            c_i[t][e] += g_i[t][e];
          }
        const double cr = a.cr[t0 + ti], ci = a.ci[t0 + ti], hh = a.h[t0 + ti];
#pragma unroll
        for (int t = 0; t < FA_NT; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double x = c_r[t][e], y = c_i[t][e];
            if (!CQ) {
              const double v = __dsub_rn(__dmul_rn(cr, x), __dmul_rn(ci, y));
              q_r[t][e] = __dsub_rn(q_r[t][e], __dmul_rn(hh, v));
            } else {
              const double vr = __dsub_rn(__dmul_rn(cr, x), __dmul_rn(ci, y));
              const double vi = __dadd_rn(__dmul_rn(cr, y), __dmul_rn(ci, x));
              q_r[t][e] = __dsub_rn(q_r[t][e], vr);
              q_i[t][e] = __dsub_rn(q_i[t][e], vi);
            }
          }
      }
#pragma unroll
      for (int t = 0; t < FA_NT; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = c0 + t * 8 + 2 * q + e;
          if (rok && col < a.nrhs) {
            a.qr[(long long)row * a.ldq + col] = q_r[t][e];
            if (CQ) a.qi[(long long)row * a.ldq + col] = q_i[t][e];
          }
        }
    }
  }
}


using PsFn = void (*)(PSArgs);
#define FB_KL_TABLE(kern, T) \
  static const T tbl[KLMAX + 1] = {nullptr, kern<1>, kern<2>, kern<3>, kern<4>, kern<5>, kern<6>, kern<7>, \
                                   kern<8>, kern<9>, kern<10>, kern<11>, kern<12>, kern<13>, kern<14>,   \
                                   kern<15>, kern<16>};

PsFn psolve_fwd_fn(int kl) {
  FB_KL_TABLE(band_psolve_fwd_kernel, PsFn)
  return tbl[kl];
}
PsFn psolve_bwd_fn(int kl, bool bulk) {
#define FB_BWD_ROW(B) {nullptr, band_psolve_bwd_kernel<1, B>, band_psolve_bwd_kernel<2, B>, band_psolve_bwd_kernel<3, B>, \
    band_psolve_bwd_kernel<4, B>, band_psolve_bwd_kernel<5, B>, band_psolve_bwd_kernel<6, B>, band_psolve_bwd_kernel<7, B>, \
    band_psolve_bwd_kernel<8, B>, band_psolve_bwd_kernel<9, B>, band_psolve_bwd_kernel<10, B>, band_psolve_bwd_kernel<11, B>, \
    band_psolve_bwd_kernel<12, B>, band_psolve_bwd_kernel<13, B>, band_psolve_bwd_kernel<14, B>, band_psolve_bwd_kernel<15, B>, \
    band_psolve_bwd_kernel<16, B>}
  static const PsFn tbl[2][KLMAX + 1] = {FB_BWD_ROW(false), FB_BWD_ROW(true)};
#undef FB_BWD_ROW
  return tbl[bulk ? 1 : 0][kl];
}

// g = A_j^-1 X_j for every partition of every item (in place)
cudaError_t psolve_launch(const PSArgs& ps, int count, cudaStream_t st) {
  const int nw = std::min(SNW, ceil_div(ps.nrhs, 32));
  const dim3 grid(ps.P * count, ceil_div(ps.nrhs, 32 * nw));  // shift fastest
  // bulk (TMA engine) staging needs 16-byte aligned right-hand-side rows
  const bool bulk = (ps.ldx & 1) == 0 && (ps.sx & 1) == 0 && ((uintptr_t)ps.xr & 15) == 0 && ((uintptr_t)ps.xi & 15) == 0;
  static DevOnce cfg[KLMAX + 1];
  if (cfg[ps.kl].first()) {  // sized for the widest CTA (SNW warps)
    cudaFuncSetAttribute(psolve_fwd_fn(ps.kl), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sweep_xring_bytes(32 * SNW, SC));
    for (int b = 0; b < 2; ++b)
      cudaFuncSetAttribute(psolve_bwd_fn(ps.kl, b != 0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sweep_xring_bytes(BNC, bwd_chunk(ps.kl)));
  }
  PSArgs a = ps;
  a.count = count;
  psolve_fwd_fn(ps.kl)<<<grid, 32 * nw, sweep_xring_bytes(32 * nw, SC), st>>>(a);
  if (ps.t4 && ((uintptr_t)ps.t4 & 15) == 0 && (ps.sa & 1) == 0) {  // kl = 16: tensor-pipe sweep
    static DevOnce c4;
    const size_t sm4 = sizeof(double) * T4_NST * T4_CHUNKD;
    if (c4.first()) cudaFuncSetAttribute(band_psolve_bwd_t4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    band_psolve_bwd_t4_kernel<<<dim3(ps.P * count * ceil_div(ps.nrhs, 8 * T4_WARPS)), 32 * T4_WARPS, sm4, st>>>(a);
    count_launch(2);
    return cudaGetLastError();
  }
  const int ncb = ps.nrhs >= BNC ? BNC : 16 * ceil_div(ps.nrhs, 16);  // two lanes per right-hand side
  psolve_bwd_fn(ps.kl, bulk)<<<dim3(ps.P * count, ceil_div(ps.nrhs, ncb)), 2 * ncb,
                               sweep_xring_bytes(ncb, bwd_chunk(ps.kl)), st>>>(a);
  count_launch(2);
  return cudaGetLastError();
}

int g_part_target = 0;

}  // namespace

void band_spike_set_part_target(int t) { g_part_target = t; }

int band_spike_parts(int n, int kl) {
  const bool dflt = g_part_target == 0 || g_part_target == 4096;
  if (g_part_target == 0) g_part_target = 4096;
  const int minsz = std::max(2 * kl + 1, std::min(64, g_part_target));
  int P = (n + g_part_target - 1) / g_part_target;
  // Wave quantisation: the sweeps run one CTA per (partition, shift, column
  // group) at 4 CTAs per SM, i.e. 592 slots on 148 SMs; with Ne = 8 or 16 shifts
  // a partition count that is a multiple of 74 fills whole waves (C4: 245 -> 222
  // partitions, -3 % per pass, profiles/r02_band_partition_sweep.txt)
  constexpr int kWave = kSMs * 4 / 8;
  if (dflt && P >= kWave) P = kWave * std::max(1, (P + kWave / 2) / kWave);
  P = std::min(P, std::max(1, n / std::max(1, minsz)));
  // every partition, the shorter last one included, keeps >= minsz rows
  while (P > 1 && n - (P - 1) * part_sz(n, P) < minsz) --P;
  return std::max(1, P);
}

bool band_spike_ok(int kl) { return kl >= 1 && kl <= KLMAX; }

// aux (per item, doubles): spikes | Dinv | F | Us [n][2kl+2] (re, im) | kl = 16: T4 (4-row DMMA fragments)
static size_t aux_spike_part(int n, int kl) {
  const int P = band_spike_parts(n, kl);
  return (size_t)4 * kl * n + (size_t)12 * kl * kl * (P > 1 ? P - 1 : 0);
}
static size_t aux_t4_doubles(int n, int kl) {
  if (kl != KLMAX) return 0;
  const int P = band_spike_parts(n, kl);
  return (size_t)(t4_steps(n, P) * P + T4_S) * T4_STEPD;  // + one chunk of slack past the last partition
}
size_t band_spike_aux_doubles(int n, int kl) {
  return aux_spike_part(n, kl) + (size_t)2 * (2 * kl + 2) * n + aux_t4_doubles(n, kl) + 64;
}
static const double2* slot_us(int n, int kl, const double* aux) {
  return reinterpret_cast<const double2*>(aux + aux_spike_part(n, kl));  // even offset: 16-byte aligned
}
static const double* slot_t4(int n, int kl, const double* aux) {
  return kl == KLMAX ? aux + aux_spike_part(n, kl) + (size_t)2 * (2 * kl + 2) * n : nullptr;
}

size_t band_spike_solve_scratch_doubles(int n, int kl, int nrhs, int count) {
  const int P = band_spike_parts(n, kl);
  // interface values [count][P-1][2kl][nrhs] + per-partition tips [count][P][2kl][nrhs], re | im
  return (size_t)count * ((P > 1 ? P - 1 : 0) + P) * 2 * kl * nrhs * 2 + 64;
}

// aux pointers of item base
static void aux_ptrs(int n, int kl, double* aux, double** sr, double** si, double** dr, double** di, double** fr,
                     double** fi) {
  const int P = band_spike_parts(n, kl);
  const size_t ns = (size_t)2 * kl * n, nd = (size_t)4 * kl * kl * (P > 1 ? P - 1 : 0),
               nf = (size_t)2 * kl * kl * (P > 1 ? P - 1 : 0);
  *sr = aux;
  *si = aux + ns;
  *dr = aux + 2 * ns;
  *di = *dr + nd;
  *fr = *di + nd;
  *fi = *fr + nf;
}

cudaError_t band_spike_factor(int count, int n, int kl, const double* zr, const double* zi, const double* far_,
                              const double* fai, const double* fbr, const double* fbi, long long ldb,
                              double* wr, double* wi, long long sw, int* ipiv, long long sp, double* aux,
                              long long sa, int* info, cudaStream_t st) {
  if (n <= 0 || count <= 0) return cudaSuccess;
  if (count > 64 || !band_spike_ok(kl)) return cudaErrorInvalidValue;
  const int P = band_spike_parts(n, kl);
  cudaError_t e;
  // zero factor arrays (entries outside the partitions are never written)
  for (int k = 0; k < count; ++k) {
    if ((e = cudaMemsetAsync(wr + k * sw, 0, sizeof(double) * band_fact_doubles(n, kl), st))) return e;
    if ((e = cudaMemsetAsync(wi + k * sw, 0, sizeof(double) * band_fact_doubles(n, kl), st))) return e;
  }
  std::vector<int> big(count, INT_MAX);
  if ((e = cudaMemcpyAsync(info, big.data(), sizeof(int) * count, cudaMemcpyHostToDevice, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;  // host vector lifetime
  PFArgs pa{};
  pa.n = n; pa.kl = kl; pa.P = P;
  for (int k = 0; k < count; ++k) {
    pa.z.r[k] = zr[k];
    pa.z.i[k] = zi[k];
  }
  pa.far_ = far_; pa.fai = fai; pa.fbr = fbr; pa.fbi = fbi; pa.ldb = ldb;
  pa.wr = wr; pa.wi = wi; pa.sw = sw; pa.ipiv = ipiv; pa.sp = sp; pa.info = info;
  band_pfactor_kernel<<<dim3(ceil_div(P, WPB), count), WPB * 32, 0, st>>>(pa);
  count_launch();
  if ((e = cudaGetLastError())) return e;
  const double2* us = slot_us(n, kl, aux);
  SOArgs so{};
  so.n = n; so.kl = kl; so.P = P; so.wr = wr; so.wi = wi; so.sw = sw;
  so.us = const_cast<double2*>(us); so.sa = sa;
  const long long tu = (long long)n * (2 * kl + 2);
  band_slot_bwd_kernel<<<dim3((int)std::min<long long>((tu + 255) / 256, 8 * kSMs), count), 256, 0, st>>>(so);
  count_launch();
  if ((e = cudaGetLastError())) return e;
  const double* t4 = slot_t4(n, kl, aux);
  if (t4) {
    T4Args ta{};
    ta.n = n; ta.P = P; ta.wr = wr; ta.wi = wi; ta.sw = sw; ta.t4 = const_cast<double*>(t4); ta.sa = sa;
    const long long tt = t4_steps(n, P) * P * T4_STEPD;
    band_t4_kernel<<<dim3((int)std::min<long long>((tt + 255) / 256, 8 * kSMs), count), 256, 0, st>>>(ta);
    count_launch();
    if ((e = cudaGetLastError())) return e;
  }
  if (P == 1) return cudaSuccess;
  double *sr, *si, *dr, *di, *fr, *fi;
  aux_ptrs(n, kl, aux, &sr, &si, &dr, &di, &fr, &fi);
  SIArgs s{};
  s.n = n; s.kl = kl; s.P = P; s.z = pa.z;
  s.far_ = far_; s.fai = fai; s.fbr = fbr; s.fbi = fbi; s.ldb = ldb;
  s.sr = sr; s.si = si; s.ss = sa;
  const long long tot = (long long)n * 2 * kl;
  band_spike_init_kernel<<<dim3((int)std::min<long long>((tot + 255) / 256, 8 * kSMs), count), 256, 0, st>>>(s);
  count_launch();
  if ((e = cudaGetLastError())) return e;
  PSArgs ps{};
  ps.n = n; ps.kl = kl; ps.P = P; ps.nrhs = 2 * kl;
  ps.wr = wr; ps.wi = wi; ps.sw = sw; ps.ipiv = ipiv; ps.sp = sp;
  ps.us = us; ps.t4 = t4; ps.sa = sa;
  ps.xr = sr; ps.xi = si; ps.ldx = 2 * kl; ps.sx = sa;
  if ((e = psolve_launch(ps, count, st))) return e;
  RFArgs rf{};
  rf.n = n; rf.kl = kl; rf.P = P;
  rf.sr = sr; rf.si = si; rf.ss = sa;
  rf.dr = dr; rf.di = di; rf.fr = fr; rf.fi = fi; rf.sa = sa; rf.info = info;
  {
    const size_t rsm = sizeof(double) * 3 * 2 * (size_t)(2 * kl) * (2 * kl);
    static DevOnce rcfg;
    if (rcfg.first())
      cudaFuncSetAttribute(band_rfactor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(double) * 3 * 2 * (2 * KLMAX) * (2 * KLMAX)));
    band_rfactor_kernel<<<count, RT, rsm, st>>>(rf);
  }
  count_launch();
  return cudaGetLastError();
}

// Sweeps, interface solve and tips of one batched solve: on return X holds the
// partition solves g and tg the tips T_j; the spike correction is left to the caller.
static cudaError_t solve_front(int count, int n, int kl, int nrhs, const double* wr, const double* wi, long long sw,
                               const int* ipiv, long long sp, const double* aux, long long sa, double* xr,
                               double* xi, long long ldx, long long sx, double* scratch, cudaStream_t st,
                               const double* yr, const double* yi, long long ldy, long long sy_, TGArgs* tg_out) {
  const int P = band_spike_parts(n, kl);
  const int chunks = ceil_div(nrhs, RS_NC);
  PSArgs ps{};
  ps.n = n; ps.kl = kl; ps.P = P; ps.nrhs = nrhs;
  ps.wr = wr; ps.wi = wi; ps.sw = sw; ps.ipiv = ipiv; ps.sp = sp;
  ps.us = slot_us(n, kl, aux);
  ps.t4 = slot_t4(n, kl, aux);
  ps.sa = sa;
  ps.xr = xr; ps.xi = xi; ps.ldx = ldx; ps.sx = sx;
  ps.fr = yr; ps.fi = yi; ps.ldf = ldy; ps.sf = sy_;
  cudaError_t e;
  if ((e = psolve_launch(ps, count, st))) return e;
  if (P == 1) return cudaSuccess;
  double *sr, *si, *dr, *di, *fr, *fi;
  aux_ptrs(n, kl, const_cast<double*>(aux), &sr, &si, &dr, &di, &fr, &fi);
  const long long sy = (long long)(P - 1) * 2 * kl * nrhs;
  RSArgs rs{};
  rs.n = n; rs.kl = kl; rs.P = P; rs.nrhs = nrhs;
  rs.sr = sr; rs.si = si; rs.ss = sa; rs.dr = dr; rs.di = di; rs.fr = fr; rs.fi = fi; rs.sa = sa;
  rs.xr = xr; rs.xi = xi; rs.ldx = ldx; rs.sx = sx;
  rs.yr = scratch; rs.yi = scratch + count * sy; rs.sy = sy;
  band_rsolve_kernel<<<dim3(count, chunks), RT, 0, st>>>(rs);
  count_launch();
  if ((e = cudaGetLastError())) return e;
  const long long w = 2 * kl, stt = (long long)P * w * nrhs;
  TGArgs tg{};
  tg.kl = kl; tg.P = P; tg.nrhs = nrhs; tg.yr = rs.yr; tg.yi = rs.yi; tg.sy = sy;
  tg.tr = scratch + 2 * count * sy; tg.ti = tg.tr + count * stt; tg.st = stt;
  band_tips_kernel<<<dim3((int)std::min<long long>(ceil_div(stt, 256), 4 * kSMs), count), 256, 0, st>>>(tg);
  count_launch();
  *tg_out = tg;
  return cudaGetLastError();
}

cudaError_t band_spike_solve(int count, int n, int kl, int nrhs, const double* wr, const double* wi, long long sw,
                             const int* ipiv, long long sp, const double* aux, long long sa, double* xr,
                             double* xi, long long ldx, long long sx, double* scratch, cudaStream_t st,
                             const double* yr, const double* yi, long long ldy, long long sy_) {
  if (n <= 0 || nrhs <= 0 || count <= 0) return cudaSuccess;
  if (!band_spike_ok(kl)) return cudaErrorInvalidValue;
  const int P = band_spike_parts(n, kl);
  cudaError_t e;
  TGArgs tg{};
  if ((e = solve_front(count, n, kl, nrhs, wr, wi, sw, ipiv, sp, aux, sa, xr, xi, ldx, sx, scratch, st, yr, yi, ldy,
                       sy_, &tg)))
    return e;
  if (P == 1) return cudaSuccess;
  double *sr, *si, *dr, *di, *fr, *fi;
  aux_ptrs(n, kl, const_cast<double*>(aux), &sr, &si, &dr, &di, &fr, &fi);
  // correction on the FP64 tensor pipe: per shift, X_j -= [V_j W_j] T_j for all
  // partitions as one strided-batch ZGEMM (K = 2kl) plus one for the shorter last
  const long long w = 2 * kl, stt = tg.st;
  const int sz = part_sz(n, P), last = n - (P - 1) * sz;
  for (int k = 0; k < count; ++k) {
    const double* ar = sr + k * sa;
    const double* ai = si + k * sa;
    const double* br = tg.tr + k * stt;
    const double* bi = tg.ti + k * stt;
    double* cr = xr + k * sx;
    double* ci = xi + k * sx;
    if ((e = gemm(1, sz, nrhs, (int)w, op_n(ar, ai, w), op_n(br, bi, nrhs), cr, ci, ldx, -1.0, 0.0, 1.0, 0.0, st,
                  nullptr, 1, P - 1, (long long)sz * w, w * nrhs, (long long)sz * ldx)))
      return e;
    const long long lo = (long long)(P - 1) * sz;
    if ((e = gemm(1, last, nrhs, (int)w, op_n(ar + lo * w, ai + lo * w, w),
                  op_n(br + (P - 1) * w * nrhs, bi + (P - 1) * w * nrhs, nrhs), cr + lo * ldx, ci + lo * ldx, ldx,
                  -1.0, 0.0, 1.0, 0.0, st)))
      return e;
  }
  return cudaSuccess;
}

// One contour pass: every item solved against the pass's right-hand side
// (yr/yi, shared: stride 0) and the quadrature terms t = 0..nterms-1
// (item[t] = which factor; mode/h/cr/ci as accumulate_terms) folded into Q.
// X is work space (it ends holding the uncorrected partition solves).
cudaError_t band_spike_solve_accumulate(int count, int n, int kl, int nrhs, const double* wr, const double* wi,
                                        long long sw, const int* ipiv, long long sp, const double* aux, long long sa,
                                        double* xr, double* xi, long long ldx, long long sx, double* scratch,
                                        cudaStream_t st, const double* yr, const double* yi, long long ldy,
                                        const AccTerms& terms, const int* item, double* qr, double* qi,
                                        long long ldq) {
  if (n <= 0 || nrhs <= 0 || count <= 0 || terms.count <= 0) return cudaSuccess;
  if (!band_spike_ok(kl) || terms.count > kMaxAccTerms) return cudaErrorInvalidValue;
  const int P = band_spike_parts(n, kl);
  cudaError_t e;
  TGArgs tg{};
  if ((e = solve_front(count, n, kl, nrhs, wr, wi, sw, ipiv, sp, aux, sa, xr, xi, ldx, sx, scratch, st, yr, yi, ldy,
                       0, &tg)))
    return e;
  if (P == 1) {  // no spikes: plain accumulation of the solves
    AccTerms t = terms;
    for (int k = 0; k < t.count; ++k) {
      t.xr[k] = xr + item[k] * sx;
      t.xi[k] = xi + item[k] * sx;
    }
    return accumulate_terms_launch(t, n, nrhs, ldx, qr, qi, ldq, st);
  }
  double *sr, *si, *dr, *di, *fr, *fi;
  aux_ptrs(n, kl, const_cast<double*>(aux), &sr, &si, &dr, &di, &fr, &fi);
  FAArgs fa{};
  fa.n = n; fa.kl = kl; fa.P = P; fa.nrhs = nrhs; fa.nterms = terms.count;
  fa.chunks = ceil_div(part_sz(n, P), FA_CHUNK);
  fa.sr = sr; fa.si = si; fa.ss = sa; fa.tr = tg.tr; fa.ti = tg.ti; fa.st = tg.st;
  fa.xr = xr; fa.xi = xi; fa.ldx = ldx; fa.sx = sx; fa.qr = qr; fa.qi = qi; fa.ldq = ldq;
  for (int k = 0; k < terms.count; ++k) {
    if (item[k] < 0 || item[k] >= count) return cudaErrorInvalidValue;
    fa.item[k] = item[k]; fa.mode[k] = terms.mode[k];
    fa.h[k] = terms.h[k]; fa.cr[k] = terms.cr[k]; fa.ci[k] = terms.ci[k];
  }
  const bool cq = terms.mode[0] != 0 && qi;
  const int KS = (2 * kl + 3) / 4;
  const size_t smem = sizeof(double) * (size_t)std::min(FA_MAXG, terms.count) * 2 * KS * FA_NT * 32;
  const dim3 grid(P * fa.chunks, ceil_div(nrhs, FA_COLS));
  static DevOnce cfg;
  if (cfg.first()) {
    const int mx = (int)(sizeof(double) * FA_MAXG * 2 * FA_KS * FA_NT * 32);
    cudaFuncSetAttribute(band_correct_accumulate_kernel<false, 384>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(band_correct_accumulate_kernel<true, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  }
  if (cq)
    band_correct_accumulate_kernel<true, 256><<<grid, 256, smem, st>>>(fa);
  else
    band_correct_accumulate_kernel<false, 384><<<grid, 384, smem, st>>>(fa);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fb
