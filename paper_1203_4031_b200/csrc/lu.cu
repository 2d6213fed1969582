// Dense shifted complex LU with partial pivoting and its multi-RHS solves.
//
// Restates feastlib's dense backend (dense.py:30-88, _DenseOps dense.py:91-117)
// as a blocked algorithm for sm_100a:
//   * shift formation S = z B - A (dense.py:97-103), planar complex;
//   * right-looking blocked LU, outer block NB = 128 (trailing update is one
//     DMMA ZGEMM with K = 128), inner sub-panels of PW = 32 columns;
//   * each sub-panel is factored by ONE kernel that keeps the panel rows
//     resident in shared memory and exchanges one (|pivot|, row, row-data)
//     record per CTA per column: through DSMEM inside a thread-block cluster
//     of <= 16 CTAs (barrier.cluster per column) when the panel fits in the
//     cluster's shared memory, else through L2 with a cooperative grid barrier;
//     argmax pivot with first-index ties (np.argmax, dense.py:41), full-row swap,
//     scaling and rank-1 update exactly as dense.py:40-49;
//   * the panel kernel also emits the 32x32 unit-lower / upper diagonal-block
//     inverses (every triangular solve downstream is then a DMMA GEMM) and the
//     panel's interchanges as a (dst, src) row list, applied to all other
//     columns by one gather/scatter kernel (no per-swap serialisation);
//   * piv[k] = row swapped with k at step k (0-based) as lu_factor; an exactly
//     zero pivot reports column k (SingularMatrixError, dense.py:42-43);
//   * the composed row permutation perm (P B)[i] = B[perm[i]] is stored with the
//     factor so the solves apply all interchanges with one parallel gather.
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm.cuh"
#include "lu.cuh"
#include "trsm.cuh"

namespace cg = cooperative_groups;

namespace fb {

namespace {

constexpr int PW = 32;         // sub-panel width (= diagonal block size of dinv)
constexpr int NB = 128;        // outer block (trailing-update K)
constexpr int PT = 128;        // threads per panel CTA
constexpr int SP = PW + 1;     // smem pitch of panel rows (conflict-free per-row access)
constexpr int RPC_CLUSTER = 384;  // max panel rows per CTA in cluster mode (~203 KB smem)
constexpr int MAX_CLUSTER = 16;
constexpr int LIST = 1 + 2 * 2 * PW;  // per-block swap list: cnt, dst[2PW], src[2PW]

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
// Row interchanges of one sub-panel, given as a (dst, src) list of <= 2*PW
// rows, applied to the columns [0, c0) u [c0+pw, n): stage the source rows of
// a 64-column strip in shared memory, then write them to their destinations.
// ---------------------------------------------------------------------------
constexpr int SW_COLS = 32;
__global__ void __launch_bounds__(256) swap_list_kernel(double* __restrict__ re, double* __restrict__ im,
                                                        long long ld, int n, int c0, int pw,
                                                        const int* __restrict__ list) {
  __shared__ double sv[2 * PW][SW_COLS][2];
  __shared__ int sdst[2 * PW], ssrc[2 * PW];
  const int cnt = list[0];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    sdst[i] = list[1 + i];
    ssrc[i] = list[1 + 2 * PW + i];
  }
  __syncthreads();
  const int ncols = n - pw;
  const int j0 = blockIdx.x * SW_COLS;
  for (int e = threadIdx.x; e < cnt * SW_COLS; e += blockDim.x) {
    int i = e / SW_COLS, jj = e % SW_COLS, j = j0 + jj;
    if (j >= ncols) continue;
    int col = j < c0 ? j : j + pw;
    long long o = (long long)ssrc[i] * ld + col;
    sv[i][jj][0] = re[o];
    sv[i][jj][1] = im[o];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < cnt * SW_COLS; e += blockDim.x) {
    int i = e / SW_COLS, jj = e % SW_COLS, j = j0 + jj;
    if (j >= ncols) continue;
    int col = j < c0 ? j : j + pw;
    long long o = (long long)sdst[i] * ld + col;
    re[o] = sv[i][jj][0];
    im[o] = sv[i][jj][1];
  }
}

// ---------------------------------------------------------------------------
// Composed permutation from the per-block lists: idx starts as identity and
// each block maps idx'[dst] = idx[src] (one CTA, idx in shared memory).
// ---------------------------------------------------------------------------
__global__ void perm_kernel(int n, const int* __restrict__ lists, int* __restrict__ perm) {
  extern __shared__ int idx[];
  __shared__ int tmp[2 * PW];
  for (int i = threadIdx.x; i < n; i += blockDim.x) idx[i] = i;
  __syncthreads();
  const int nblk = ceil_div(n, PW);
  for (int b = 0; b < nblk; ++b) {
    const int* L = lists + (size_t)b * LIST;
    const int cnt = L[0];
    if (threadIdx.x < cnt) tmp[threadIdx.x] = idx[L[1 + 2 * PW + threadIdx.x]];
    __syncthreads();
    if (threadIdx.x < cnt) idx[L[1 + threadIdx.x]] = tmp[threadIdx.x];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = idx[i];
}

// out[i][j] = in[perm[i]][j] (gather = 1) or out[perm[i]][j] = in[i][j] (scatter)
__global__ void permute_rows_kernel(int n, int m, const int* __restrict__ perm, int gather,
                                    const double* __restrict__ ir, const double* __restrict__ ii,
                                    long long ldi, double* __restrict__ orr, double* __restrict__ oi,
                                    long long ldo) {
  long long total = (long long)n * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    int p = perm[i];
    if (gather) {
      orr[i * ldo + j] = ir[(long long)p * ldi + j];
      oi[i * ldo + j] = ii[(long long)p * ldi + j];
    } else {
      orr[(long long)p * ldo + j] = ir[i * ldi + j];
      oi[(long long)p * ldo + j] = ii[i * ldi + j];
    }
  }
}

// ---------------------------------------------------------------------------
// Sub-panel factorization.
// ---------------------------------------------------------------------------
struct PanelArgs {
  double* re;
  double* im;
  long long ld;
  int n, c0, pw, rpc;
  int* piv;
  int* info;
  double* xrec;   // GRID mode: [2][G][2 + 2*PW] (val, row, data), in L2
  double* xrowr;  // GRID mode: [2][2*PW] copy of row rj
  double* linv;   // [2 planes][PW][PW] inverse of unit-lower diagonal block
  double* uinv;   // [2 planes][PW][PW] inverse of upper diagonal block
  int* list;      // [LIST] swap list of this sub-panel
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

enum { MODE_GRID = 0, MODE_CLUSTER = 1 };

template <int MODE>
__global__ void __launch_bounds__(PT) panel_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  int G, g;
  if (MODE == MODE_CLUSTER) {
    G = (int)cg::this_cluster().num_blocks();
    g = (int)cg::this_cluster().block_rank();
  } else {
    G = gridDim.x;
    g = blockIdx.x;
  }
  const int rbeg = a.c0 + g * a.rpc;
  const int rend = min(a.n, rbeg + a.rpc);
  const int cnt = max(0, rend - rbeg);
  constexpr int REC = 2 + 2 * PW;
  double* sre = sm;                       // [rpc][SP]
  double* sim = sm + a.rpc * SP;          // [rpc][SP]
  double* prow = sim + a.rpc * SP;        // [2*PW] pivot row
  double* rrow = prow + 2 * PW;           // [2*PW] old row rj
  double* lrec = rrow + 2 * PW;           // CLUSTER: [2][REC] own record
  double* lrj = lrec + 2 * REC;           // CLUSTER: [2][2*PW] own copy of row rj
  __shared__ Best red[PT / 32];
  __shared__ int s_gw;
  __shared__ int s_piv[PW];

  for (int e = tid; e < cnt * PW; e += PT) {
    int lr = e / PW, c = e % PW;
    long long off = (long long)(rbeg + lr) * a.ld + a.c0 + c;
    bool ok = c < a.pw;
    sre[lr * SP + c] = ok ? a.re[off] : 0.0;
    sim[lr * SP + c] = ok ? a.im[off] : 0.0;
  }
  __syncthreads();
  const int owner_rows = a.rpc;

  for (int j = 0; j < a.pw; ++j) {
    const int rj = a.c0 + j;
    const int par = j & 1;
    // 1. local argmax of |a[r, j]| over own rows r >= rj
    Best b{-1.0, 0x7fffffff};
    for (int lr = tid; lr < cnt; lr += PT) {
      int gr = rbeg + lr;
      if (gr >= rj) b = better(b, Best{cabs_(sre[lr * SP + j], sim[lr * SP + j]), gr});
    }
    b = block_best(b, red);
    const bool own_best = b.v >= 0.0 && b.r >= rbeg && b.r < rend;
    const bool own_rj = rj >= rbeg && rj < rend;
    // 2. publish the record (and the owner's copy of row rj), 3. barrier
    if (MODE == MODE_CLUSTER) {
      double* rec = lrec + par * REC;
      if (tid == 0) {
        rec[0] = b.v;
        rec[1] = (double)b.r;
      }
      if (own_best) {
        int lr = b.r - rbeg;
        for (int c = tid; c < PW; c += PT) {
          rec[2 + c] = sre[lr * SP + c];
          rec[2 + PW + c] = sim[lr * SP + c];
        }
      }
      if (own_rj) {
        int lr = rj - rbeg;
        for (int c = tid; c < PW; c += PT) {
          lrj[par * 2 * PW + c] = sre[lr * SP + c];
          lrj[par * 2 * PW + PW + c] = sim[lr * SP + c];
        }
      }
      cg::this_cluster().sync();
    } else {
      double* rec = a.xrec + ((size_t)par * G + g) * REC;
      if (tid == 0) {
        __stcg(rec, b.v);
        __stcg(rec + 1, (double)b.r);
      }
      if (own_best) {
        int lr = b.r - rbeg;
        for (int c = tid; c < PW; c += PT) {
          __stcg(rec + 2 + c, sre[lr * SP + c]);
          __stcg(rec + 2 + PW + c, sim[lr * SP + c]);
        }
      }
      if (own_rj) {
        int lr = rj - rbeg;
        for (int c = tid; c < PW; c += PT) {
          __stcg(a.xrowr + par * 2 * PW + c, sre[lr * SP + c]);
          __stcg(a.xrowr + par * 2 * PW + PW + c, sim[lr * SP + c]);
        }
      }
      if (G > 1) {
        __threadfence();
        cg::this_grid().sync();
      } else {
        __syncthreads();
      }
    }
    // 4. global winner
    Best w{-1.0, 0x7fffffff};
    int wg = 0;
    for (int q = tid; q < G; q += PT) {
      Best t;
      if (MODE == MODE_CLUSTER) {
        const double* rr = cg::this_cluster().map_shared_rank(lrec + par * REC, q);
        t = Best{rr[0], (int)rr[1]};
      } else {
        const double* rr = a.xrec + ((size_t)par * G + q) * REC;
        t = Best{__ldcg(rr), (int)__ldcg(rr + 1)};
      }
      Best nb = better(w, t);
      if (nb.r != w.r || nb.v != w.v) wg = q;
      w = nb;
    }
    Best wb = block_best(w, red);
    if (w.v == wb.v && w.r == wb.r && w.v >= 0.0) s_gw = wg;  // unique row -> unique writer
    const int rj_owner = (rj - a.c0) / owner_rows;
    for (int c = tid; c < 2 * PW; c += PT) {
      if (MODE == MODE_CLUSTER)
        rrow[c] = cg::this_cluster().map_shared_rank(lrj + par * 2 * PW, rj_owner)[c];
      else
        rrow[c] = __ldcg(a.xrowr + par * 2 * PW + c);
    }
    __syncthreads();
    const int gw = s_gw;
    for (int c = tid; c < 2 * PW; c += PT) {
      if (MODE == MODE_CLUSTER)
        prow[c] = cg::this_cluster().map_shared_rank(lrec + par * REC, gw)[2 + c];
      else
        prow[c] = __ldcg(a.xrec + ((size_t)par * G + gw) * REC + 2 + c);
    }
    int p = wb.r;
    const bool zero = !(wb.v > 0.0);
    if (zero) {
      p = rj;
      if (g == 0 && tid == 0) atomicMin(a.info, rj + 1);
    }
    if (tid == 0) s_piv[j] = p;
    if (g == 0 && tid == 0) a.piv[rj] = p;
    __syncthreads();
    // 5. swap rows p <-> rj (full panel width), then scale and rank-1 update
    if (p != rj) {
      if (p >= rbeg && p < rend) {
        int lr = p - rbeg;
        for (int c = tid; c < PW; c += PT) {
          sre[lr * SP + c] = rrow[c];
          sim[lr * SP + c] = rrow[PW + c];
        }
      }
      if (own_rj) {
        int lr = rj - rbeg;
        for (int c = tid; c < PW; c += PT) {
          sre[lr * SP + c] = prow[c];
          sim[lr * SP + c] = prow[PW + c];
        }
      }
      __syncthreads();
    }
    if (!zero) {
      const double pr = prow[j], pi = prow[PW + j];
      const double den = pr * pr + pi * pi;
      const double ir = pr / den, ii = -pi / den;
      for (int lr = tid; lr < cnt; lr += PT) {
        if (rbeg + lr <= rj) continue;
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
  if (MODE == MODE_CLUSTER) cg::this_cluster().sync();  // remote readers done before exit

  // write back
  for (int e = tid; e < cnt * a.pw; e += PT) {
    int lr = e / a.pw, c = e % a.pw;
    long long off = (long long)(rbeg + lr) * a.ld + a.c0 + c;
    a.re[off] = sre[lr * SP + c];
    a.im[off] = sim[lr * SP + c];
  }
  if (g != 0) return;
  // swap list of this sub-panel (dst row <- content of src row)
  if (tid < 32) {
    const int t = tid;
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
  // diagonal-block inverses
  if (tid < PW) {
    const int c = tid;
    double xr[PW], xi[PW];
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

int g_grid_max_blocks = 0;
bool g_cluster_ok = false;
bool g_cluster_probed = false;

size_t panel_smem(int rpc) { return sizeof(double) * (2 * (size_t)rpc * SP + 4 * PW + 2 * (2 + 2 * PW) + 4 * PW); }

}  // namespace

size_t zgetrf_scratch_bytes(int n) {
  (void)n;
  const int Gmax = 4 * kSMs;
  return sizeof(double) * (2 * (size_t)Gmax * (2 + 2 * PW) + 2 * 2 * PW) + 256;
}

// Factor side storage, in doubles: [nblk][4][PW][PW] diagonal inverses (L re/im,
// U re/im), then perm[n] ints, then nblk swap lists.
// ... then the per-block sweep operators G (trsm.cu) of the fused solves.
static size_t lists_doubles(int n) { return ((size_t)ceil_div(n, PW) * LIST + 1) / 2 + 2; }
size_t dinv_doubles(int n) {
  size_t nblk = ceil_div(n, PW);
  return nblk * 4 * PW * PW + ceil_div(n, 2) + lists_doubles(n) + gmat_doubles(n);
}
const int* factor_perm(const double* dinv, int n) {
  return reinterpret_cast<const int*>(dinv + (size_t)ceil_div(n, PW) * 4 * PW * PW);
}
static int* factor_lists(double* dinv, int n) {
  return reinterpret_cast<int*>(dinv + (size_t)ceil_div(n, PW) * 4 * PW * PW + ceil_div(n, 2));
}
const double* factor_gmat(const double* dinv, int n) {
  return dinv + (size_t)ceil_div(n, PW) * 4 * PW * PW + ceil_div(n, 2) + lists_doubles(n);
}

cudaError_t shift_launch(int n, double zr, double zi, const double* are, const double* aim,
                         long long lda, const double* bre, const double* bim, long long ldb,
                         double* sre, double* sim, long long lds, cudaStream_t st) {
  long long total = (long long)n * n;
  int blocks = (int)std::min<long long>((total + 255) / 256, 8 * kSMs);
  shift_kernel<<<blocks, 256, 0, st>>>(n, zr, zi, are, aim, lda, bre, bim, ldb, sre, sim, lds);
  count_launch();
  return cudaGetLastError();
}

cudaError_t permute_rows_launch(int n, int m, const int* perm, int gather, const double* ir,
                                const double* ii, long long ldi, double* orr, double* oi,
                                long long ldo, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  long long total = (long long)n * m;
  int blocks = (int)std::min<long long>((total + 255) / 256, 16 * kSMs);
  permute_rows_kernel<<<blocks, 256, 0, st>>>(n, m, perm, gather, ir, ii, ldi, orr, oi, ldo);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t panel_launch(double* re, double* im, long long ld, int n, int c0, int pw, int* piv,
                                int* info, char* scratch, double* linv, double* uinv, int* list,
                                cudaStream_t st) {
  const int rows = n - c0;
  const int smem_cap = 210 * 1024;
  PanelArgs a;
  a.re = re; a.im = im; a.ld = ld; a.n = n; a.c0 = c0; a.pw = pw;
  a.piv = piv; a.info = info; a.linv = linv; a.uinv = uinv; a.list = list;
  double* d = reinterpret_cast<double*>(scratch);
  const int Gmax = 4 * kSMs;
  a.xrec = d;
  a.xrowr = d + 2 * (size_t)Gmax * (2 + 2 * PW);
  if (!g_cluster_probed) {
    g_cluster_probed = true;
    cudaFuncSetAttribute(panel_kernel<MODE_CLUSTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap);
    cudaFuncSetAttribute(panel_kernel<MODE_CLUSTER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(panel_kernel<MODE_GRID>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = MAX_CLUSTER;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(MAX_CLUSTER);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = panel_smem(RPC_CLUSTER);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, panel_kernel<MODE_CLUSTER>, &cfg);
    g_cluster_ok = (e == cudaSuccess && clusters >= 1);
    cudaGetLastError();
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, panel_kernel<MODE_GRID>, PT, panel_smem(128));
    g_grid_max_blocks = std::max(1, nb);
  }
  count_launch();
  if (rows <= RPC_CLUSTER || (g_cluster_ok && rows <= MAX_CLUSTER * RPC_CLUSTER)) {
    int G = std::max(1, std::min(MAX_CLUSTER, ceil_div(rows, RPC_CLUSTER)));
    // keep CTA 0 holding the whole diagonal block, and use more CTAs for tall panels
    if (rows > 2 * PW) G = std::max(G, std::min(MAX_CLUSTER, ceil_div(rows, 256)));
    G = std::max(1, std::min(G, rows / PW));
    int rpc = ceil_div(rows, G);
    G = ceil_div(rows, rpc);
    a.rpc = rpc;
    size_t smem = panel_smem(rpc);
    if (G == 1) {
      panel_kernel<MODE_GRID><<<1, PT, smem, st>>>(a);
      return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, panel_kernel<MODE_CLUSTER>, a);
  }
  int G = ceil_div(rows, 128);
  G = std::max(1, std::min(G, rows / PW));
  G = std::min(G, g_grid_max_blocks * kSMs);
  int rpc = ceil_div(rows, G);
  G = ceil_div(rows, rpc);
  a.rpc = rpc;
  size_t smem = panel_smem(rpc);
  if ((int)smem > smem_cap) return cudaErrorInvalidConfiguration;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)panel_kernel<MODE_GRID>, dim3(G), dim3(PT), args, smem, st);
}

static cudaError_t swap_list_launch(double* re, double* im, long long ld, int n, int c0, int pw,
                                    const int* list, cudaStream_t st) {
  int ncols = n - pw;
  if (ncols <= 0) return cudaSuccess;
  swap_list_kernel<<<ceil_div(ncols, SW_COLS), 256, 0, st>>>(re, im, ld, n, c0, pw, list);
  count_launch();
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
  int* lists = factor_lists(dinv, n);
  for (int k = 0; k < n; k += NB) {
    const int nb = std::min(NB, n - k);
    for (int s = 0; s < nb; s += PW) {
      const int c0 = k + s, pw = std::min(PW, nb - s), blk = c0 / PW;
      int* list = lists + (size_t)blk * LIST;
      e = panel_launch(re, im, ld, n, c0, pw, piv, info, scratch, L(blk), U(blk), list, st);
      if (e != cudaSuccess) return e;
      if ((e = swap_list_launch(re, im, ld, n, c0, pw, list, st))) return e;
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
  // composed permutation for the solves
  size_t psmem = sizeof(int) * (size_t)n;
  static bool pcfg = false;
  if (!pcfg) {
    cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    pcfg = true;
  }
  if (psmem > 200 * 1024) return cudaErrorInvalidValue;
  perm_kernel<<<1, 256, psmem, st>>>(n, lists, const_cast<int*>(factor_perm(dinv, n)));
  count_launch();
  if ((e = cudaGetLastError())) return e;
  return gmat_launch(n, re, im, ld, dinv, const_cast<double*>(factor_gmat(dinv, n)), st);
}

// Solve op(A) X = B in place for X (n x nrhs planar, ldx) from zgetrf output.
// adjoint = 0: A X = B (dense.py:62-74); adjoint = 1: A^H X = B (dense.py:75-87).
// tmp: n*nrhs*2 doubles of scratch for the row permutation.
cudaError_t zgetrs(int n, int nrhs, const double* re, const double* im, long long ld, const int* piv,
                   const double* dinv, int adjoint, double* xr, double* xi, long long ldx, double* tmp,
                   cudaStream_t st) {
  cudaError_t e;
  (void)piv;
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int nblk = ceil_div(n, PW);
  const int* perm = factor_perm(dinv, n);
  double* tr = tmp;
  double* ti = tmp + (size_t)n * nrhs;
  auto L = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW; };
  auto U = [&](int blk) { return dinv + (size_t)blk * 4 * PW * PW + 2 * PW * PW; };
  auto row = [&](const double* p, int r, int c) { return p + (long long)r * ld + c; };
  static const bool blocked = getenv("FB_SOLVE_BLOCKED") != nullptr;  // A/B switch for tests
  if (!blocked) {
    const double* gm = factor_gmat(dinv, n);
    if (!adjoint) {
      if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
      if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
      if ((e = permute_rows_launch(n, nrhs, perm, 1, tr, ti, nrhs, xr, xi, ldx, st))) return e;
      if ((e = sweep_launch(0, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st))) return e;
      return sweep_launch(1, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st);
    }
    if ((e = sweep_launch(2, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st))) return e;
    if ((e = sweep_launch(3, n, nrhs, re, im, ld, dinv, gm, xr, xi, ldx, st))) return e;
    if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    return permute_rows_launch(n, nrhs, perm, 0, tr, ti, nrhs, xr, xi, ldx, st);
  }
  if (!adjoint) {
    // X <- P X (one gather through the scratch copy)
    if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = permute_rows_launch(n, nrhs, perm, 1, tr, ti, nrhs, xr, xi, ldx, st))) return e;
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
  // A^H = U^H L^H P: forward with U^H, backward with L^H, then X <- P^T X
  for (int b = 0; b < nblk; ++b) {
    const int r0 = b * PW, pw = std::min(PW, n - r0);
    double* x0r = xr + (long long)r0 * ldx;
    double* x0i = xi + (long long)r0 * ldx;
    if ((e = gemm(1, pw, nrhs, pw, op_c(U(b), U(b) + PW * PW, PW), op_n(x0r, x0i, ldx), x0r, x0i, ldx,
                  1.0, 0.0, 0.0, 0.0, st)))
      return e;
    const int below = n - r0 - pw;
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
    if (r0 > 0 && (e = gemm(1, r0, nrhs, pw, op_c(row(re, r0, 0), row(im, r0, 0), ld),
                            op_n(x0r, x0i, ldx), xr, xi, ldx, -1.0, 0.0, 1.0, 0.0, st)))
      return e;
  }
  if ((e = cudaMemcpy2DAsync(tr, nrhs * 8, xr, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpy2DAsync(ti, nrhs * 8, xi, ldx * 8, nrhs * 8, n, cudaMemcpyDeviceToDevice, st))) return e;
  return permute_rows_launch(n, nrhs, perm, 0, tr, ti, nrhs, xr, xi, ldx, st);
}

}  // namespace fb
