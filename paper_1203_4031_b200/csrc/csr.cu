// CSR backend helpers (feast_scsr / feast_hcsr, sparse.py:430-517).
//
//   csr_spmm       _csr_block_matvec sparse.py:156-169 (multiply_a / multiply_b,
//                  sparse.py:454-462): Y = M X for a full-pattern CSR M and a
//                  row-major N x m block X, real or planar complex on both sides
//   permute_rows   dst(i, :) = src(perm(i), :) -- moves solve right-hand sides
//                  into and out of the bandwidth-reducing order the shifted
//                  systems are factored in
//
// Both are HBM-bound.  One warp covers 32 consecutive columns of one row, so
// every X row segment is a coalesced 256-byte read; the row's (index, value)
// stream is a warp-uniform broadcast load.  Products are accumulated in the
// pattern's column order, the order of np.add.reduceat in the reference.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "csr.cuh"

namespace fb {

namespace {

constexpr int kRowsPerCta = 8;

template <bool ACPLX, bool XCPLX>
__global__ void __launch_bounds__(256) csr_spmm_kernel(int n, int m, const long long* __restrict__ indptr,
                                                       const long long* __restrict__ indices,
                                                       const double* __restrict__ vr,
                                                       const double* __restrict__ vi,
                                                       const double* __restrict__ xr,
                                                       const double* __restrict__ xi, long long ldx,
                                                       double* __restrict__ yr, double* __restrict__ yi,
                                                       long long ldy, const long long* __restrict__ order) {
  const int slot = blockIdx.x * kRowsPerCta + threadIdx.y;
  const int col = blockIdx.y * 32 + threadIdx.x;
  if (slot >= n) return;
  // rows visited in a bandwidth-reducing order: rows processed together share
  // neighbours, so the X rows they gather are re-read from L2, not HBM
  const long long row = order ? order[slot] : slot;
  const long long k0 = indptr[row], k1 = indptr[row + 1];
  if (col >= m) return;
  double ar = 0.0, ai = 0.0;
  auto fma_term = [&](double a, double b, double p, double q) {
    if (XCPLX) {
      if (ACPLX) {
        ar += a * p - b * q;
        ai += a * q + b * p;
      } else {
        ar += a * p;
        ai += a * q;
      }
    } else {
      ar += a * p;
      if (ACPLX) ai += b * p;
    }
  };
  long long k = k0;
  // four entries' index/value loads, then their four X gathers, in flight
  // together (the chain index -> X row is otherwise one latency per entry);
  // the sum is still taken in pattern order
  for (; k + 4 <= k1; k += 4) {
    long long j[4];
    double a[4], b[4], p[4], q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      j[u] = indices[k + u];
      a[u] = vr[k + u];
      b[u] = ACPLX ? vi[k + u] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      p[u] = xr[j[u] * ldx + col];
      q[u] = XCPLX ? xi[j[u] * ldx + col] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) fma_term(a[u], b[u], p[u], q[u]);
  }
  for (; k < k1; ++k) {
    const long long j = indices[k];
    fma_term(vr[k], ACPLX ? vi[k] : 0.0, xr[j * ldx + col], XCPLX ? xi[j * ldx + col] : 0.0);
  }
  yr[row * ldy + col] = ar;
  if (ACPLX || XCPLX) yi[row * ldy + col] = ai;
}

// 16-byte moves when both strides and the column count allow it
template <int V>
__global__ void __launch_bounds__(256) gather_rows_kernel(int n, int mv, const long long* __restrict__ perm,
                                                           const double* __restrict__ sr,
                                                           const double* __restrict__ si, long long lds,
                                                           double* __restrict__ dr, double* __restrict__ di,
                                                           long long ldd) {
  using VT = typename std::conditional<V == 2, double2, double>::type;
  const int row = blockIdx.x * kRowsPerCta + threadIdx.y;
  if (row >= n) return;
  const long long src = perm[row];
  for (int c = threadIdx.x + blockIdx.y * 32; c < mv; c += 32 * gridDim.y) {
    reinterpret_cast<VT*>(dr + (long long)row * ldd)[c] = reinterpret_cast<const VT*>(sr + src * lds)[c];
    if (si) reinterpret_cast<VT*>(di + (long long)row * ldd)[c] = reinterpret_cast<const VT*>(si + src * lds)[c];
  }
}

}  // namespace

cudaError_t csr_spmm_launch(int n, int m, const long long* indptr, const long long* indices, const double* vr,
                            const double* vi, const double* xr, const double* xi, long long ldx, double* yr,
                            double* yi, long long ldy, const long long* order, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  const bool acplx = vi != nullptr, xcplx = xi != nullptr;
  if ((acplx || xcplx) && yi == nullptr) return cudaErrorInvalidValue;
  count_launch();
  dim3 grid(ceil_div(n, kRowsPerCta), ceil_div(m, 32)), block(32, kRowsPerCta);
  if (acplx && xcplx)
    csr_spmm_kernel<true, true><<<grid, block, 0, st>>>(n, m, indptr, indices, vr, vi, xr, xi, ldx, yr, yi, ldy, order);
  else if (acplx)
    csr_spmm_kernel<true, false><<<grid, block, 0, st>>>(n, m, indptr, indices, vr, vi, xr, xi, ldx, yr, yi, ldy, order);
  else if (xcplx)
    csr_spmm_kernel<false, true><<<grid, block, 0, st>>>(n, m, indptr, indices, vr, vi, xr, xi, ldx, yr, yi, ldy, order);
  else
    csr_spmm_kernel<false, false><<<grid, block, 0, st>>>(n, m, indptr, indices, vr, vi, xr, xi, ldx, yr, yi,
                                                          ldy, order);
  return cudaGetLastError();
}

cudaError_t gather_rows_launch(int n, int m, const long long* perm, const double* sr, const double* si,
                                long long lds, double* dr, double* di, long long ldd, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  if ((si == nullptr) != (di == nullptr)) return cudaErrorInvalidValue;
  count_launch();
  const bool vec = (m % 2 == 0) && (lds % 2 == 0) && (ldd % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(sr) | reinterpret_cast<uintptr_t>(dr) |
                     reinterpret_cast<uintptr_t>(si) | reinterpret_cast<uintptr_t>(di)) % 16 == 0);
  const int mv = vec ? m / 2 : m;
  dim3 grid(ceil_div(n, kRowsPerCta), ceil_div(mv, 32) > 4 ? 4 : ceil_div(mv, 32)), block(32, kRowsPerCta);
  if (vec)
    gather_rows_kernel<2><<<grid, block, 0, st>>>(n, mv, perm, sr, si, lds, dr, di, ldd);
  else
    gather_rows_kernel<1><<<grid, block, 0, st>>>(n, mv, perm, sr, si, lds, dr, di, ldd);
  return cudaGetLastError();
}

}  // namespace fb

// ---- lockstep BiCGStab (_bicgstab, sparse.py:354-391) ---------------------------------------
//
// All right-hand-side columns iterate together; each keeps the reference's
// own scalars (rho, alpha, omega) and stop tests.  Column reductions are
// two-stage and fixed-order (per-CTA partials, then one thread per column
// sums them), so results do not depend on scheduling.  Vectors are planar
// complex, row-major n x m with leading dimension ld.
namespace fb {
namespace {

constexpr int kRedRows = 8;   // row groups per reduction CTA (x 32 columns)

struct Cplx {
  double r, i;
};
__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ Cplx cdiv(Cplx a, Cplx b) {
  // numpy's complex division (Smith's algorithm), as the reference's scalars use
  if (fabs(b.r) >= fabs(b.i)) {
    if (b.r == 0.0 && b.i == 0.0) return {a.r / fabs(b.r), a.i / fabs(b.i)};
    const double rat = b.i / b.r, scl = 1.0 / (b.r + b.i * rat);
    return {(a.r + a.i * rat) * scl, (a.i - a.r * rat) * scl};
  }
  const double rat = b.r / b.i, scl = 1.0 / (b.i + b.r * rat);
  return {(a.r * rat + a.i) * scl, (a.i * rat - a.r) * scl};
}

// partial[blk][c] = sum over this CTA's rows of conj(a(r, c)) * b(r, c)
__global__ void __launch_bounds__(256) bicg_colred_kernel(int n, int m, const double* __restrict__ ar,
                                                          const double* __restrict__ ai,
                                                          const double* __restrict__ br,
                                                          const double* __restrict__ bi, long long ld,
                                                          const int* __restrict__ status,
                                                          double* __restrict__ part) {
  __shared__ double sr[kRedRows][33], si[kRedRows][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  double accr = 0.0, acci = 0.0;
  if (c < m && status[c] == 0) {
    for (int r = blockIdx.y * kRedRows + threadIdx.y; r < n; r += gridDim.y * kRedRows) {
      const long long o = (long long)r * ld + c;
      const double xr = ar[o], xi = ai[o], yr = br[o], yi = bi[o];
      accr += xr * yr + xi * yi;
      acci += xr * yi - xi * yr;
    }
  }
  sr[threadIdx.y][threadIdx.x] = accr;
  si[threadIdx.y][threadIdx.x] = acci;
  __syncthreads();
  if (threadIdx.y == 0 && c < m) {
    double tr = 0.0, ti = 0.0;
    for (int k = 0; k < kRedRows; ++k) {
      tr += sr[k][threadIdx.x];
      ti += si[k][threadIdx.x];
    }
    part[2 * ((long long)blockIdx.y * m + c)] = tr;
    part[2 * ((long long)blockIdx.y * m + c) + 1] = ti;
  }
}

// per-column state: st[c*12 + ...] = rho(2) alpha(2) omega(2) beta(2) rho1(2) bnorm tol*bnorm
enum { S_RHO = 0, S_ALPHA = 2, S_OMEGA = 4, S_BETA = 6, S_RHO1 = 8, S_BNORM = 10, S_TOLB = 11, S_W = 12 };

// step 0: init (bnorm from part = |b|^2); 1: rho1, beta; 2: alpha; 3: |s| test;
// 4: omega (part = (t,t), part2 = (t,s)); 5: |r| test, iteration count
__global__ void bicg_scalar_kernel(int step, int m, int nparts, const double* __restrict__ part,
                                   const double* __restrict__ part2, double tol, int maxiter,
                                   double* __restrict__ st, int* __restrict__ status, int* __restrict__ iters) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  if (step == 4 && status[c] == 2) {   // x already took alpha * phat: column final
    status[c] = 1;
    return;
  }
  if (step != 0 && status[c] != 0) return;
  Cplx s1 = {0.0, 0.0}, s2 = {0.0, 0.0};
  for (int k = 0; k < nparts; ++k) {
    s1.r += part[2 * ((long long)k * m + c)];
    s1.i += part[2 * ((long long)k * m + c) + 1];
    if (part2) {
      s2.r += part2[2 * ((long long)k * m + c)];
      s2.i += part2[2 * ((long long)k * m + c) + 1];
    }
  }
  double* S = st + (long long)c * S_W;
  switch (step) {
    case 0: {
      const double bn = sqrt(s1.r);
      S[S_BNORM] = bn;
      S[S_TOLB] = tol * bn;
      S[S_RHO] = S[S_ALPHA] = S[S_OMEGA] = 1.0;
      S[S_RHO + 1] = S[S_ALPHA + 1] = S[S_OMEGA + 1] = 0.0;
      status[c] = bn == 0.0 ? 1 : 0;  // zero right-hand side: x = 0
      iters[c] = 0;
      break;
    }
    case 1: {
      if (s1.r == 0.0 && s1.i == 0.0) { status[c] = -1; break; }
      const Cplx rho = {S[S_RHO], S[S_RHO + 1]}, al = {S[S_ALPHA], S[S_ALPHA + 1]},
                 om = {S[S_OMEGA], S[S_OMEGA + 1]};
      const Cplx beta = cmul(cdiv(s1, rho), cdiv(al, om));
      S[S_BETA] = beta.r; S[S_BETA + 1] = beta.i;
      S[S_RHO1] = s1.r; S[S_RHO1 + 1] = s1.i;
      break;
    }
    case 2: {
      if (s1.r == 0.0 && s1.i == 0.0) { status[c] = -2; break; }
      const Cplx al = cdiv({S[S_RHO1], S[S_RHO1 + 1]}, s1);
      S[S_ALPHA] = al.r; S[S_ALPHA + 1] = al.i;
      break;
    }
    case 3:
      if (sqrt(s1.r) <= S[S_TOLB]) status[c] = 2;   // x += alpha * phat, then done
      break;
    case 4: {
      if (s1.r == 0.0 && s1.i == 0.0) { status[c] = -3; break; }
      const Cplx om = cdiv(s2, s1);
      S[S_OMEGA] = om.r; S[S_OMEGA + 1] = om.i;
      break;
    }
    case 5: {
      if (sqrt(s1.r) <= S[S_TOLB]) { status[c] = 1; break; }
      S[S_RHO] = S[S_RHO1]; S[S_RHO + 1] = S[S_RHO1 + 1];
      if (++iters[c] >= maxiter) status[c] = -4;
      break;
    }
  }
}

// elementwise steps over active columns (planar complex, row-major, ld):
//  0: x = 0, r = b, rhat = b, p = v = 0          (all columns)
//  1: p = r + beta (p - omega v); phat = p / d
//  2: s = r - alpha v
//  3: status 2: x += alpha phat (-> 1); active: shat = s / d
//  4: x = x + alpha phat + omega shat; r = s - omega t
struct BicgVecs {
  double *xr, *xi, *rr, *ri, *hr, *hi, *pr, *pi, *vr, *vi, *sr, *si, *tr, *ti, *qr, *qi, *wr, *wi;
  // q = phat, w = shat, h = rhat
};

__global__ void __launch_bounds__(256) bicg_update_kernel(int step, int n, int m, long long ld, BicgVecs V,
                                                          const double* __restrict__ br,
                                                          const double* __restrict__ bi, long long ldb,
                                                          const double* __restrict__ dr,
                                                          const double* __restrict__ di,
                                                          const double* __restrict__ st,
                                                          int* __restrict__ status) {
  const int c = blockIdx.y * 32 + threadIdx.x;
  const int row = blockIdx.x * 8 + threadIdx.y;
  if (c >= m || row >= n) return;
  const int stc = status[c];
  const long long o = (long long)row * ld + c;
  const double* S = st + (long long)c * S_W;
  if (step == 0) {
    const double b0 = br[(long long)row * ldb + c], b1 = bi ? bi[(long long)row * ldb + c] : 0.0;
    V.xr[o] = 0.0; V.xi[o] = 0.0;
    V.rr[o] = b0; V.ri[o] = b1;
    V.hr[o] = b0; V.hi[o] = b1;
    V.pr[o] = 0.0; V.pi[o] = 0.0;
    V.vr[o] = 0.0; V.vi[o] = 0.0;
    return;
  }
  if (step == 3) {
    const Cplx al = {S[S_ALPHA], S[S_ALPHA + 1]};
    if (stc == 2) {
      const Cplx a = cmul(al, {V.qr[o], V.qi[o]});
      V.xr[o] += a.r; V.xi[o] += a.i;
    } else if (stc == 0) {
      const Cplx w = cdiv({V.sr[o], V.si[o]}, {dr[row], di[row]});
      V.wr[o] = w.r; V.wi[o] = w.i;
    }
    return;
  }
  if (stc != 0) return;
  if (step == 1) {
    const Cplx beta = {S[S_BETA], S[S_BETA + 1]}, om = {S[S_OMEGA], S[S_OMEGA + 1]};
    const Cplx ov = cmul(om, {V.vr[o], V.vi[o]});
    const Cplx bp = cmul(beta, {V.pr[o] - ov.r, V.pi[o] - ov.i});
    const Cplx p = {V.rr[o] + bp.r, V.ri[o] + bp.i};
    V.pr[o] = p.r; V.pi[o] = p.i;
    const Cplx q = cdiv(p, {dr[row], di[row]});
    V.qr[o] = q.r; V.qi[o] = q.i;
  } else if (step == 2) {
    const Cplx av = cmul({S[S_ALPHA], S[S_ALPHA + 1]}, {V.vr[o], V.vi[o]});
    V.sr[o] = V.rr[o] - av.r; V.si[o] = V.ri[o] - av.i;
  } else if (step == 4) {
    const Cplx aq = cmul({S[S_ALPHA], S[S_ALPHA + 1]}, {V.qr[o], V.qi[o]});
    const Cplx om = {S[S_OMEGA], S[S_OMEGA + 1]};
    const Cplx ow = cmul(om, {V.wr[o], V.wi[o]});
    V.xr[o] = (V.xr[o] + aq.r) + ow.r; V.xi[o] = (V.xi[o] + aq.i) + ow.i;
    const Cplx ot = cmul(om, {V.tr[o], V.ti[o]});
    V.rr[o] = V.sr[o] - ot.r; V.ri[o] = V.si[o] - ot.i;
  }
}

__global__ void count_active_kernel(int m, const int* __restrict__ status, int* __restrict__ out) {
  // out[0] = active columns, out[1] = first failed column's code (0 if none)
  int act = 0, fail = 0;
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    act += status[c] == 0 || status[c] == 2;
    if (status[c] < 0 && fail == 0) fail = status[c];
  }
  for (int o = 16; o; o >>= 1) {
    act += __shfl_xor_sync(0xffffffffu, act, o);
    const int f = __shfl_xor_sync(0xffffffffu, fail, o);
    if (fail == 0) fail = f;
  }
  if (threadIdx.x == 0) { out[0] = act; out[1] = fail; }
}

}  // namespace

size_t bicgstab_workspace_doubles(int n, int m, long long ld) {
  const int parts = bicgstab_parts(n);
  return (size_t)16 * n * ld + (size_t)m * S_W + (size_t)4 * parts * m;
}

int bicgstab_parts(int n) {
  const int p = ceil_div(n, kRedRows * 64);
  return p < 1 ? 1 : (p > 2 * kSMs ? 2 * kSMs : p);
}

// Solve S X = B for all m columns; S = (indptr, indices, s_re/s_im) full CSR,
// d = its diagonal (zeros replaced by 1).  X overwrites B's storage is not
// assumed: b and x are separate planar blocks.  Returns via flags[0] the
// number of still-active columns and flags[1] the first failure code
// (-1 rho, -2 rhat.v, -3 t.t breakdown, -4 maxiter); the host polls these.
cudaError_t bicgstab_launch(int phase, int n, int m, const long long* indptr, const long long* indices,
                            const double* s_re, const double* s_im, const double* d_re, const double* d_im,
                            const double* b_re, const double* b_im, long long ldb, double* x_re, double* x_im,
                            long long ldx, double tol, int maxiter, int iters, double* work, long long ld,
                            int* istate, const long long* order, cudaStream_t st) {
  // work layout: 8 planar vectors (r rhat p v s t phat shat), then state, then partials
  const long long plane = (long long)n * ld;
  BicgVecs V;
  double* w = work;
  auto take = [&](double*& re, double*& im) { re = w; im = w + plane; w += 2 * plane; };
  V.xr = x_re; V.xi = x_im;
  take(V.rr, V.ri); take(V.hr, V.hi); take(V.pr, V.pi); take(V.vr, V.vi);
  take(V.sr, V.si); take(V.tr, V.ti); take(V.qr, V.qi); take(V.wr, V.wi);
  double* stt = w;
  double* part = stt + (size_t)m * S_W;
  double* part2 = part + (size_t)2 * bicgstab_parts(n) * m;
  int* status = istate;
  int* itc = istate + m;
  int* flags = istate + 2 * m;
  const int parts = bicgstab_parts(n);
  const dim3 rgrid(ceil_div(m, 32), parts), rblk(32, kRedRows);
  const dim3 ugrid(ceil_div(n, 8), ceil_div(m, 32)), ublk(32, 8);
  const int sblk = 128, sgrid = ceil_div(m, sblk);
  if (ldx != ld) return cudaErrorInvalidValue;
  if (phase == 0) {
    count_launch(3);
    cudaMemsetAsync(status, 0, sizeof(int) * m, st);
    bicg_update_kernel<<<ugrid, ublk, 0, st>>>(0, n, m, ld, V, b_re, b_im, ldb, d_re, d_im, stt, status);
    bicg_colred_kernel<<<rgrid, rblk, 0, st>>>(n, m, V.rr, V.ri, V.rr, V.ri, ld, status, part);
    bicg_scalar_kernel<<<sgrid, sblk, 0, st>>>(0, m, parts, part, nullptr, tol, maxiter, stt, status, itc);
    return cudaGetLastError();
  }
  auto run_iters = [&](cudaStream_t q) {
  for (int it = 0; it < iters; ++it) {
    bicg_colred_kernel<<<rgrid, rblk, 0, q>>>(n, m, V.hr, V.hi, V.rr, V.ri, ld, status, part);
    bicg_scalar_kernel<<<sgrid, sblk, 0, q>>>(1, m, parts, part, nullptr, tol, maxiter, stt, status, itc);
    bicg_update_kernel<<<ugrid, ublk, 0, q>>>(1, n, m, ld, V, b_re, b_im, ldb, d_re, d_im, stt, status);
    csr_spmm_kernel<true, true><<<dim3(ceil_div(n, kRowsPerCta), ceil_div(m, 32)), dim3(32, kRowsPerCta), 0, q>>>(
        n, m, indptr, indices, s_re, s_im, V.qr, V.qi, ld, V.vr, V.vi, ld, order);
    bicg_colred_kernel<<<rgrid, rblk, 0, q>>>(n, m, V.hr, V.hi, V.vr, V.vi, ld, status, part);
    bicg_scalar_kernel<<<sgrid, sblk, 0, q>>>(2, m, parts, part, nullptr, tol, maxiter, stt, status, itc);
    bicg_update_kernel<<<ugrid, ublk, 0, q>>>(2, n, m, ld, V, b_re, b_im, ldb, d_re, d_im, stt, status);
    bicg_colred_kernel<<<rgrid, rblk, 0, q>>>(n, m, V.sr, V.si, V.sr, V.si, ld, status, part);
    bicg_scalar_kernel<<<sgrid, sblk, 0, q>>>(3, m, parts, part, nullptr, tol, maxiter, stt, status, itc);
    bicg_update_kernel<<<ugrid, ublk, 0, q>>>(3, n, m, ld, V, b_re, b_im, ldb, d_re, d_im, stt, status);
    // columns that met the |s| test are final (status 2 -> 1)
    csr_spmm_kernel<true, true><<<dim3(ceil_div(n, kRowsPerCta), ceil_div(m, 32)), dim3(32, kRowsPerCta), 0, q>>>(
        n, m, indptr, indices, s_re, s_im, V.wr, V.wi, ld, V.tr, V.ti, ld, order);
    bicg_colred_kernel<<<rgrid, rblk, 0, q>>>(n, m, V.tr, V.ti, V.tr, V.ti, ld, status, part);
    bicg_colred_kernel<<<rgrid, rblk, 0, q>>>(n, m, V.tr, V.ti, V.sr, V.si, ld, status, part2);
    bicg_scalar_kernel<<<sgrid, sblk, 0, q>>>(4, m, parts, part, part2, tol, maxiter, stt, status, itc);
    bicg_update_kernel<<<ugrid, ublk, 0, q>>>(4, n, m, ld, V, b_re, b_im, ldb, d_re, d_im, stt, status);
    bicg_colred_kernel<<<rgrid, rblk, 0, q>>>(n, m, V.rr, V.ri, V.rr, V.ri, ld, status, part);
    bicg_scalar_kernel<<<sgrid, sblk, 0, q>>>(5, m, parts, part, nullptr, tol, maxiter, stt, status, itc);
  }
  };
  count_launch(16 * iters);
  // The `iters`-iteration chunk is replayed from a CUDA graph captured on a
  // private stream (16 launches per iteration; capture needs a non-legacy
  // stream, torch's current stream is usually the legacy one).  Cached by the
  // full argument tuple, so a hit replays exactly the same launches.
  static const bool use_graph = [] {
    const char* e = getenv("FB_BICG_GRAPH");
    return !(e && e[0] == '0');
  }();
  if (!use_graph || iters == 0) {
    run_iters(st);
  } else {
    struct Key {
      const void* p[14];
      long long l[3];
      double tol;
      int i[5];
    } key;
    memset(&key, 0, sizeof(key));
    const void* ps[14] = {indptr, indices, s_re, s_im, d_re, d_im, b_re, b_im, x_re, x_im, work, istate, st, order};
    memcpy(key.p, ps, sizeof(ps));
    key.l[0] = ldb; key.l[1] = ldx; key.l[2] = ld;
    key.tol = tol;
    key.i[0] = n; key.i[1] = m; key.i[2] = maxiter; key.i[3] = iters;
    int cur_dev = 0;
    cudaGetDevice(&cur_dev);
    key.i[4] = cur_dev;  // graphs and the capture stream belong to one device
    struct Entry {
      Key k;
      cudaGraphExec_t exec;
    };
    static std::vector<Entry> cache;
    static std::mutex mu;
    static cudaStream_t caps[64] = {};
    cudaStream_t& cap = caps[cur_dev & 63];
    std::lock_guard<std::mutex> lock(mu);
    cudaGraphExec_t exec = nullptr;
    for (auto& e : cache)
      if (!memcmp(&e.k, &key, sizeof(Key))) exec = e.exec;
    if (!exec) {
      if (!cap) {
        cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return e;
      run_iters(cap);
      e = cudaStreamEndCapture(cap, &g);
      if (e != cudaSuccess) return e;
      e = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return e;
      if (cache.size() >= 256) {
        cudaGraphExecDestroy(cache.front().exec);
        cache.erase(cache.begin());
      }
      cache.push_back({key, exec});
    }
    cudaError_t e = cudaGraphLaunch(exec, st);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  count_active_kernel<<<1, 32, 0, st>>>(m, status, flags);
  return cudaGetLastError();
}

}  // namespace fb
