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

// ---- partition solve (direct): one warp per (partition, 32 columns, shift) ----
struct PSArgs {
  int n, kl, P, nrhs;
  const double *wr, *wi;
  long long sw;
  const int* ipiv;
  long long sp;
  double *xr, *xi;
  long long ldx, sx;
  // forward sweep input (nullptr: in place from x); fi == nullptr: real input;
  // sf = 0: one right-hand-side block shared by every item (the pass's Y)
  const double *fr, *fi;
  long long ldf, sf;
};

template <int KL>
__global__ void __launch_bounds__(WPB * 32) band_psolve_kernel(PSArgs a) {
  constexpr int KV = 2 * KL, LW = 3 * KL + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int part = blockIdx.x * WPB + wid, chunk = blockIdx.y, k = blockIdx.z;
  if (part >= a.P) return;
  const int col = chunk * 32 + lane;
  const bool on = col < a.nrhs;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const double* Wr = a.wr + k * a.sw;
  const double* Wi = a.wi + k * a.sw;
  const int* ipiv = a.ipiv + k * a.sp;
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  auto ld = [&](int r, double& vr, double& vi) {
    if (on && r < hi) {
      const long long o = (long long)r * a.ldx + col;
      vr = Xr[o];
      vi = Xi[o];
    } else {
      vr = vi = 0.0;
    }
  };
  // forward: pivots interleaved with unit L (rows j..j+KL live)
  double wr_[KL + 1], wi_[KL + 1];
#pragma unroll
  for (int i = 0; i <= KL; ++i) ld(lo + i, wr_[i], wi_[i]);
  for (int j = lo; j < hi; ++j) {
    const int p = ipiv[j] - j;
    if (p) {
#pragma unroll
      for (int i = 1; i <= KL; ++i)
        if (i == p) {
          const double tr = wr_[0], ti = wi_[0];
          wr_[0] = wr_[i];
          wi_[0] = wi_[i];
          wr_[i] = tr;
          wi_[i] = ti;
        }
    }
    const double x0r = wr_[0], x0i = wi_[0];
    const double* lr = Wr + (long long)j * LW + KV + 1;
    const double* li = Wi + (long long)j * LW + KV + 1;
#pragma unroll
    for (int i = 0; i < KL; ++i) {  // multipliers beyond the partition are stored as 0
      const double ar = __ldg(lr + i), ai = __ldg(li + i);
      wr_[1 + i] -= ar * x0r - ai * x0i;
      wi_[1 + i] -= ar * x0i + ai * x0r;
    }
    if (on) {
      const long long o = (long long)j * a.ldx + col;
      Xr[o] = x0r;
      Xi[o] = x0i;
    }
#pragma unroll
    for (int i = 0; i < KL; ++i) {
      wr_[i] = wr_[i + 1];
      wi_[i] = wi_[i + 1];
    }
    ld(j + KL + 1, wr_[KL], wi_[KL]);
  }
  // backward: x_j = y_j / U_jj, then y[j-KV..j-1] -= U[., j] x_j (rows j-KV..j live)
  double ur_[KV + 1], ui_[KV + 1];
  auto ldb = [&](int r, double& vr, double& vi) {
    if (on && r >= lo) {
      const long long o = (long long)r * a.ldx + col;
      vr = Xr[o];
      vi = Xi[o];
    } else {
      vr = vi = 0.0;
    }
  };
#pragma unroll
  for (int i = 0; i <= KV; ++i) ldb(hi - 1 - KV + i, ur_[i], ui_[i]);
  for (int j = hi - 1; j >= lo; --j) {
    const double* cr = Wr + (long long)j * LW;
    const double* ci = Wi + (long long)j * LW;
    const double dr = __ldg(cr + KV), di = __ldg(ci + KV);
    const double den = dr * dr + di * di;
    const double yr = ur_[KV], yi = ui_[KV];
    const double qr = (yr * dr + yi * di) / den, qi = (yi * dr - yr * di) / den;
#pragma unroll
    for (int i = 0; i < KV; ++i) {  // U entries above the partition are stored as 0
      const double br = __ldg(cr + i), bi = __ldg(ci + i);
      ur_[i] -= br * qr - bi * qi;
      ui_[i] -= br * qi + bi * qr;
    }
    if (on) {
      const long long o = (long long)j * a.ldx + col;
      Xr[o] = qr;
      Xi[o] = qi;
    }
#pragma unroll
    for (int i = KV; i > 0; --i) {
      ur_[i] = ur_[i - 1];
      ui_[i] = ui_[i - 1];
    }
    ldb(j - 1 - KV, ur_[0], ui_[0]);
  }
}

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

// ---- correction x_j = g_j - V_j x_{j+1}^t - W_j x_{j-1}^b -----------------------
struct CKArgs {
  int n, kl, P, nrhs;
  const double *sr, *si;
  long long ss;
  const double *yr, *yi;
  long long sy;
  double *xr, *xi;
  long long ldx, sx;
};

template <int KL>
__global__ void __launch_bounds__(WPB * 32) band_correct_kernel(CKArgs a) {
  constexpr int W2 = 2 * KL;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int part = blockIdx.x * WPB + wid, chunk = blockIdx.y, k = blockIdx.z;
  if (part >= a.P) return;
  const int col = chunk * 32 + lane;
  if (col >= a.nrhs) return;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const double* Sr = a.sr + k * a.ss;
  const double* Si = a.si + k * a.ss;
  const double* Yr = a.yr + k * a.sy;
  const double* Yi = a.yi + k * a.sy;
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  double tr[W2], ti[W2];  // (x_{j+1}^t, x_{j-1}^b)
#pragma unroll
  for (int q = 0; q < KL; ++q) {
    const bool nx = part + 1 < a.P, pv = part > 0;
    const long long on = ((long long)part * W2 + KL + q) * a.nrhs + col;        // y_part[kl + q]
    const long long op = ((long long)(part - 1) * W2 + q) * a.nrhs + col;       // y_{part-1}[q]
    tr[q] = nx ? Yr[on] : 0.0;
    ti[q] = nx ? Yi[on] : 0.0;
    tr[KL + q] = pv ? Yr[op] : 0.0;
    ti[KL + q] = pv ? Yi[op] : 0.0;
  }
  for (int r = lo; r < hi; ++r) {
    const double* sr = Sr + (long long)r * W2;
    const double* si = Si + (long long)r * W2;
    double ar = 0.0, ai = 0.0;
#pragma unroll
    for (int q = 0; q < W2; ++q) {
      const double vr = __ldg(sr + q), vi = __ldg(si + q);
      ar += vr * tr[q] - vi * ti[q];
      ai += vr * ti[q] + vi * tr[q];
    }
    const long long o = (long long)r * a.ldx + col;
    Xr[o] -= ar;
    Xi[o] -= ai;
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

// ---- staged partition solves: one CTA per (partition, column block, shift) -------
// All warps of a CTA share the factor columns, staged through shared memory in
// chunks of TC columns by cp.async (double-buffered) with re/im interleaved so
// one LDS.128 feeds a complex multiply-add; each thread keeps its right-hand
// side column's active rows in a register window and the next QD rows in a
// prefetch queue (the global load of a row entering the window was issued QD
// steps earlier).  Forward (pivots + unit L) and backward (U) are separate
// kernels so each keeps its own register window.
constexpr int TC = 32;     // rows per staged chunk (correction)
constexpr int SNW = 3;     // warps per CTA (96 right-hand sides)

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

// Sweeps stage SC rows per chunk: the factor columns of the chunk's rows and,
// for every thread's column, the SC right-hand-side rows that will ENTER the
// register window during the chunk, one chunk ahead by cp.async (no register
// queue; the load of a row is issued ~SC steps of the whole CTA before use).
constexpr int SC = 12;   // forward sweep (4 CTAs per SM)
constexpr int SCB = 12;  // backward sweep chunk (4 CTAs per SM at <= 168 registers)
size_t sweep_xring_bytes(int nt, int sc = SC) { return sizeof(double) * 2 * sc * 2 * (size_t)nt; }

template <int KL>
__global__ void __launch_bounds__(SNW * 32, 4) band_psolve_fwd_kernel(PSArgs a) {
  constexpr int KV = 2 * KL, LW = 3 * KL + 1;
  const int part = blockIdx.x, k = blockIdx.z, tid = threadIdx.x, nt = blockDim.x;
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
  extern __shared__ double sx[];  // [2 buf][SC rows][2 planes][nt]
  __shared__ double2 sl[2][SC][KL];  // multipliers (re, im) of column j
  __shared__ int spv[2][SC];
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
    double* xb = sx + (size_t)buf * SC * 2 * nt;
#pragma unroll
    for (int r = 0; r < SC; ++r) {
      const int row = xbase + c * SC + r;
      const bool ok = on && row < hi;
      const long long o = ok ? (long long)row * ldf + col : 0;
      cp_async8(xb + (r * 2) * nt + tid, Fr + o, ok);
      cp_async8(xb + (r * 2 + 1) * nt + tid, Fi ? Fi + o : Fr + o, ok && Fi != nullptr);
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
  const int nch = (hi - lo + SC - 1) / SC;
  stage(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      stage(buf ^ 1, c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int j0 = lo + c * SC, jn = min(SC, hi - j0);
    const double* xb = sx + (size_t)buf * SC * 2 * nt;
#pragma unroll 1
    for (int jj = 0; jj < jn; ++jj) {
      const int j = j0 + jj;
      const int p = spv[buf][jj] - j;
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
        const long long o = (long long)j * a.ldx + col;
        Xr[o] = x0r;
        Xi[o] = x0i;
      }
      wr_[KL] = xb[(jj * 2) * nt + tid];
      wi_[KL] = xb[(jj * 2 + 1) * nt + tid];
    }
    __syncthreads();
  }
}

// Backward sweep: one thread per right-hand side holds rows j-KV..j in
// registers; the U column (re, im interleaved, 1/U_jj computed per chunk)
// and the rows entering the window come from shared memory.
template <int KL>
__global__ void __launch_bounds__(SNW * 32, 4) band_psolve_bwd_kernel(PSArgs a) {
  constexpr int KV = 2 * KL, LW = 3 * KL + 1;
  const int part = blockIdx.x, k = blockIdx.z, tid = threadIdx.x, nt = blockDim.x;
  const int col = blockIdx.y * nt + tid;
  const bool on = col < a.nrhs;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const double* Wr = a.wr + k * a.sw;
  const double* Wi = a.wi + k * a.sw;
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  extern __shared__ double sx[];         // [2 buf][SCB rows][2 planes][nt]
  __shared__ double2 su[2][SCB][KV + 1];  // U column j (rows j-KV..j); slot KV <- 1/U_jj
  const int xtop = hi - 2 - KV;          // row entering the window at step hi-1
  auto stage = [&](int buf, int c) {
    const int j1 = hi - 1 - c * SCB;
    for (int e = tid; e < SCB * (KV + 1); e += nt) {
      const int jj = e / (KV + 1), i = e % (KV + 1), j = j1 - jj;
      const bool ok = j >= lo;
      const long long o = ok ? (long long)j * LW + i : 0;
      cp_async8(&su[buf][jj][i].x, Wr + o, ok);
      cp_async8(&su[buf][jj][i].y, Wi + o, ok);
    }
    double* xb = sx + (size_t)buf * SCB * 2 * nt;
#pragma unroll
    for (int r = 0; r < SCB; ++r) {
      const int row = xtop - c * SCB - r;
      const bool ok = on && row >= lo;
      const long long o = ok ? (long long)row * a.ldx + col : 0;
      cp_async8(xb + (r * 2) * nt + tid, Xr + o, ok);
      cp_async8(xb + (r * 2 + 1) * nt + tid, Xi + o, ok);
    }
    cp_async_commit();
  };
  double wr_[KV + 1], wi_[KV + 1];  // wr_[t] = row j-KV+t
#pragma unroll
  for (int t = 0; t <= KV; ++t) {
    const int r = hi - 1 - KV + t;
    wr_[t] = wi_[t] = 0.0;
    if (on && r >= lo) {
      const long long o = (long long)r * a.ldx + col;
      wr_[t] = Xr[o];
      wi_[t] = Xi[o];
    }
  }
  const int nch = (hi - lo + SCB - 1) / SCB;
  stage(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      stage(buf ^ 1, c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    for (int jj = tid; jj < SCB; jj += nt) {
      const double2 d = su[buf][jj][KV];
      const double den = d.x * d.x + d.y * d.y;
      su[buf][jj][KV] = den > 0.0 ? make_double2(d.x / den, -d.y / den) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int j1 = hi - 1 - c * SCB, jn = min(SCB, j1 - lo + 1);
    const double* xb = sx + (size_t)buf * SCB * 2 * nt;
#pragma unroll 1
    for (int jj = 0; jj < jn; ++jj) {
      const int j = j1 - jj;
      const double2 dv = su[buf][jj][KV];
      const double qr = wr_[KV] * dv.x - wi_[KV] * dv.y, qi = wr_[KV] * dv.y + wi_[KV] * dv.x;
      // rows j-KV+t -= U(., j) x_j, written one slot up (the window slides)
#pragma unroll
      for (int t = KV - 1; t >= 0; --t) {
        if (t % 8 == 7) asm volatile("" ::: "memory");
        const double2 u = su[buf][jj][t];
        wr_[t + 1] = fma(-u.x, qr, fma(u.y, qi, wr_[t]));
        wi_[t + 1] = fma(-u.x, qi, fma(-u.y, qr, wi_[t]));
      }
      if (on) {
        const long long o = (long long)j * a.ldx + col;
        Xr[o] = qr;
        Xi[o] = qi;
      }
      wr_[0] = xb[(jj * 2) * nt + tid];
      wi_[0] = xb[(jj * 2 + 1) * nt + tid];
    }
    __syncthreads();
  }
}

// correction with the spike rows staged through shared memory (cp.async 16 B)
template <int KL>
__global__ void __launch_bounds__(SNW * 32) band_correct2_kernel(CKArgs a) {
  constexpr int W2 = 2 * KL;
  const int part = blockIdx.x, k = blockIdx.z, tid = threadIdx.x;
  const int col = blockIdx.y * blockDim.x + tid;
  const bool on = col < a.nrhs;
  const int lo = part_lo(part, a.n, a.P), hi = part_lo(part + 1, a.n, a.P);
  const double* Sr = a.sr + k * a.ss;
  const double* Si = a.si + k * a.ss;
  const double* Yr = a.yr + k * a.sy;
  const double* Yi = a.yi + k * a.sy;
  double* Xr = a.xr + k * a.sx;
  double* Xi = a.xi + k * a.sx;
  __shared__ __align__(16) double ss[2][2][TC][W2];
  double tr[W2], ti[W2];  // (x_{j+1}^t, x_{j-1}^b) of this column
#pragma unroll
  for (int q = 0; q < KL; ++q) {
    const bool nx = part + 1 < a.P && on, pv = part > 0 && on;
    const long long on_ = ((long long)part * W2 + KL + q) * a.nrhs + col;
    const long long op = ((long long)(part - 1) * W2 + q) * a.nrhs + col;
    tr[q] = nx ? Yr[on_] : 0.0;
    ti[q] = nx ? Yi[on_] : 0.0;
    tr[KL + q] = pv ? Yr[op] : 0.0;
    ti[KL + q] = pv ? Yi[op] : 0.0;
  }
  const bool v16 = (W2 % 2) == 0;
  auto stage = [&](int buf, int r0) {
    if (v16) {
      for (int e = tid; e < TC * W2 / 2; e += blockDim.x) {
        const int rr = e / (W2 / 2), q = (e % (W2 / 2)) * 2, r = r0 + rr;
        const int ok = r < hi ? 16 : 0;
        const long long o = ok ? (long long)r * W2 + q : 0;
        cp_async16(&ss[buf][0][rr][q], Sr + o, ok);
        cp_async16(&ss[buf][1][rr][q], Si + o, ok);
      }
    }
    cp_async_commit();
  };
  stage(0, lo);
  int buf = 0;
  for (int r0 = lo; r0 < hi; r0 += TC, buf ^= 1) {
    if (r0 + TC < hi) {
      stage(buf ^ 1, r0 + TC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int rn = min(TC, hi - r0);
    if (on) {
      constexpr int G8 = 8;
      for (int g0 = 0; g0 < rn; g0 += G8) {
        double xr8[G8], xi8[G8];
#pragma unroll
        for (int u = 0; u < G8; ++u) {
          const bool ok = g0 + u < rn;
          const long long o = (long long)(r0 + g0 + u) * a.ldx + col;
          xr8[u] = ok ? __ldcs(Xr + o) : 0.0;
          xi8[u] = ok ? __ldcs(Xi + o) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < G8; ++u) {
          const int rr = g0 + u;
          if (rr >= rn) break;
          double ar = 0.0, ai = 0.0;
#pragma unroll
          for (int q = 0; q < W2; ++q) {
            const double vr = ss[buf][0][rr][q], vi = ss[buf][1][rr][q];
            ar += vr * tr[q] - vi * ti[q];
            ai += vr * ti[q] + vi * tr[q];
          }
          const long long o = (long long)(r0 + rr) * a.ldx + col;
          __stcs(Xr + o, xr8[u] - ar);
          __stcs(Xi + o, xi8[u] - ai);
        }
      }
    }
    __syncthreads();
  }
}

using PsFn = void (*)(PSArgs);
using CkFn = void (*)(CKArgs);
#define FB_KL_TABLE(kern, T) \
  static const T tbl[KLMAX + 1] = {nullptr, kern<1>, kern<2>, kern<3>, kern<4>, kern<5>, kern<6>, kern<7>, \
                                   kern<8>, kern<9>, kern<10>, kern<11>, kern<12>, kern<13>, kern<14>,   \
                                   kern<15>, kern<16>};

PsFn psolve_fwd_fn(int kl) {
  FB_KL_TABLE(band_psolve_fwd_kernel, PsFn)
  return tbl[kl];
}
PsFn psolve_bwd_fn(int kl) {
  FB_KL_TABLE(band_psolve_bwd_kernel, PsFn)
  return tbl[kl];
}
CkFn correct_fn(int kl) {
  FB_KL_TABLE(band_correct2_kernel, CkFn)
  return tbl[kl];
}

// g = A_j^-1 X_j for every partition of every item (in place)
cudaError_t psolve_launch(const PSArgs& ps, int count, cudaStream_t st) {
  const int nw = std::min(SNW, ceil_div(ps.nrhs, 32));
  const dim3 grid(ps.P, ceil_div(ps.nrhs, 32 * nw), count);
  static bool cfg[KLMAX + 1] = {};
  if (!cfg[ps.kl]) {  // sized for the widest CTA (SNW warps)
    cudaFuncSetAttribute(psolve_fwd_fn(ps.kl), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sweep_xring_bytes(32 * SNW, SC));
    cudaFuncSetAttribute(psolve_bwd_fn(ps.kl), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sweep_xring_bytes(32 * SNW, SCB));
    cfg[ps.kl] = true;
  }
  psolve_fwd_fn(ps.kl)<<<grid, 32 * nw, sweep_xring_bytes(32 * nw, SC), st>>>(ps);
  psolve_bwd_fn(ps.kl)<<<grid, 32 * nw, sweep_xring_bytes(32 * nw, SCB), st>>>(ps);
  count_launch(2);
  return cudaGetLastError();
}

int g_part_target = 0;

}  // namespace

void band_spike_set_part_target(int t) { g_part_target = t; }

int band_spike_parts(int n, int kl) {
  if (g_part_target == 0) {
    const char* e = getenv("FB_BAND_PART");
    g_part_target = e && atoi(e) > 0 ? atoi(e) : 4096;
  }
  const int minsz = std::max(2 * kl + 1, std::min(64, g_part_target));
  int P = (n + g_part_target - 1) / g_part_target;
  P = std::min(P, std::max(1, n / std::max(1, minsz)));
  // every partition, the shorter last one included, keeps >= minsz rows
  while (P > 1 && n - (P - 1) * part_sz(n, P) < minsz) --P;
  return std::max(1, P);
}

bool band_spike_ok(int kl) { return kl >= 1 && kl <= KLMAX; }

size_t band_spike_aux_doubles(int n, int kl) {
  const int P = band_spike_parts(n, kl);
  return (size_t)4 * kl * n + (size_t)12 * kl * kl * (P > 1 ? P - 1 : 0) + 64;
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
  ps.xr = sr; ps.xi = si; ps.ldx = 2 * kl; ps.sx = sa;
  if ((e = psolve_launch(ps, count, st))) return e;
  RFArgs rf{};
  rf.n = n; rf.kl = kl; rf.P = P;
  rf.sr = sr; rf.si = si; rf.ss = sa;
  rf.dr = dr; rf.di = di; rf.fr = fr; rf.fi = fi; rf.sa = sa; rf.info = info;
  {
    const size_t rsm = sizeof(double) * 3 * 2 * (size_t)(2 * kl) * (2 * kl);
    static bool rcfg = false;
    if (!rcfg) {
      cudaFuncSetAttribute(band_rfactor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(double) * 3 * 2 * (2 * KLMAX) * (2 * KLMAX)));
      rcfg = true;
    }
    band_rfactor_kernel<<<count, RT, rsm, st>>>(rf);
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t band_spike_solve(int count, int n, int kl, int nrhs, const double* wr, const double* wi, long long sw,
                             const int* ipiv, long long sp, const double* aux, long long sa, double* xr,
                             double* xi, long long ldx, long long sx, double* scratch, cudaStream_t st,
                             const double* yr, const double* yi, long long ldy, long long sy_) {
  if (n <= 0 || nrhs <= 0 || count <= 0) return cudaSuccess;
  if (!band_spike_ok(kl)) return cudaErrorInvalidValue;
  const int P = band_spike_parts(n, kl);
  const int chunks = ceil_div(nrhs, RS_NC);
  PSArgs ps{};
  ps.n = n; ps.kl = kl; ps.P = P; ps.nrhs = nrhs;
  ps.wr = wr; ps.wi = wi; ps.sw = sw; ps.ipiv = ipiv; ps.sp = sp;
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
  if (getenv("FB_BAND_CORRECT_SIMT")) {
    CKArgs ck{};
    ck.n = n; ck.kl = kl; ck.P = P; ck.nrhs = nrhs;
    ck.sr = sr; ck.si = si; ck.ss = sa; ck.yr = rs.yr; ck.yi = rs.yi; ck.sy = sy;
    ck.xr = xr; ck.xi = xi; ck.ldx = ldx; ck.sx = sx;
    const int nw = std::min(SNW, ceil_div(nrhs, 32));
    correct_fn(kl)<<<dim3(P, ceil_div(nrhs, 32 * nw), count), 32 * nw, 0, st>>>(ck);
    count_launch();
    return cudaGetLastError();
  }
  // correction on the FP64 tensor pipe: per shift, X_j -= [V_j W_j] T_j for all
  // partitions as one strided-batch ZGEMM (K = 2kl) plus one for the shorter last
  const long long w = 2 * kl, stt = (long long)P * w * nrhs;
  TGArgs tg{};
  tg.kl = kl; tg.P = P; tg.nrhs = nrhs; tg.yr = rs.yr; tg.yi = rs.yi; tg.sy = sy;
  tg.tr = scratch + 2 * count * sy; tg.ti = tg.tr + count * stt; tg.st = stt;
  band_tips_kernel<<<dim3((int)std::min<long long>(ceil_div(stt, 256), 4 * kSMs), count), 256, 0, st>>>(tg);
  count_launch();
  if ((e = cudaGetLastError())) return e;
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

}  // namespace fb
