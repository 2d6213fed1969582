// TMA-fed FP64 tensor-core ZGEMM for the bulk trailing update of the blocked LU,
//     A22 -= L21 * U12        (dense.py:49, the rank-1 np.outer update, blocked K = 256)
// for all shifts of a batch, and for the pending-row updates of the blocked
// triangular sweeps, X_pend -= M(pend, block) X_block (dense.py:62-87; M^H for the
// adjoint sweeps: template CONJT, B tiles from a second set of maps over X).  Every operand is a sub-block of the SAME strided
// batch of factor matrices (planar re / im, row-major, leading dimension ld),
// so four 3-D tensor maps (plane x {A box, B box}) describe the whole batch
// once per factorization and the kernel addresses tiles by coordinates:
//   * one elected thread issues cp.async.bulk.tensor (SASS UTMALDG) for the
//     A tile (64 rows x 16 k, one box per plane) and the B tile (16 k x 64
//     columns, four 16-column boxes per plane) of a stage onto the stage's
//     "full" mbarrier (32 KB of transaction bytes); the 8 consumer warps free
//     a stage through its "empty" mbarrier -- no per-thread staging
//     instructions or address registers (the cp.async kernel spends 16
//     LDGSTS + their address math per thread and k-tile);
//   * tiles land in shared memory with the 128-byte swizzle; the k index of a
//     DMMA step is permuted (lane quarter q takes k = base + (q & 1) + 4 (q >> 1))
//     so that both the A fragments (rows x k) and the B fragments (k x columns)
//     read all 32 banks in the minimum two wavefronts;
//   * 8 warps of 32 x 16, complex as 4 real DMMA 8x8x4 on planar operands, the
//     product accumulated from zero and added to C once (one rounding per
//     element), C loads issued together before the adds.
// Out-of-range rows / columns of a tile are either zero-filled by the TMA
// (outside the matrix) or belong to other valid entries of the factor whose
// products are never stored; the K range must be a multiple of 16.
#include <cuda.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm.cuh"

namespace fb {

namespace {

constexpr int TM = 64, TN = 64, TK = 16, TST = 3;
constexpr int A_BYTES = TM * TK * 8, B_BYTES = TK * TN * 8;      // per plane
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;             // 32 KB

struct TmaArgs {
  int m, n, k;              // C is m x n, K = k (multiple of 16)
  int arow, acol;           // A(0, 0) = M[arow][acol]
  int brow, bcol;           // B(0, 0) = M[brow][bcol]
  double *cre, *cim;        // C(0, 0) of batch item 0
  long long ldc, sc;        // C leading dimension and batch stride
  int ncol0;                // first column of this launch (a 32-wide launch covers a ragged tail)
};

__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, int c0, int c1, int c2, void* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
          "r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// CONJT: the A operand is the conjugate TRANSPOSE of a block of the tensor (the adjoint sweeps'
// M^H).  Its tile is ONE un-swizzled box per plane, 16 k-rows of 64 tensor columns ([k][row],
// 512-byte rows), so a stage is the same 10 bulk loads as the direct form; the A fragments then
// read 4 wavefronts instead of 2 (the four k of a step share their banks), well inside the
// shared-memory time the DMMAs leave.
// TNW = 64: the 8-warp CTA (two per SM).  TNW = 32: four warps on a 64 x 32 tile (three CTAs per
// SM) for a ragged tail of at most 32 columns -- M0 = 152 is 2 x 64 + 24, and a third 64-wide
// tile would spend a quarter of the update's tensor time on columns that do not exist.
template <bool CONJT, int TNW>
__global__ void __launch_bounds__(TNW * 4, TNW == 64 ? 2 : 3)
zgemm_tma_kernel(const __grid_constant__ CUtensorMap map_are, const __grid_constant__ CUtensorMap map_aim,
                 const __grid_constant__ CUtensorMap map_bre, const __grid_constant__ CUtensorMap map_bim,
                 const TmaArgs p) {
  extern __shared__ __align__(16) unsigned char tsm[];
  constexpr int NWC = TNW / 16, NTH = 2 * NWC * 32;           // column groups, threads
  constexpr int BB = TK * TNW * 8, SB = 2 * A_BYTES + 2 * BB;  // B plane and stage bytes
  __shared__ __align__(8) unsigned long long full[TST], empty[TST];
  __shared__ volatile unsigned sink[NTH / 32];
  // the 128-byte swizzle is a function of the shared-memory ADDRESS: the tiles must start on a
  // 1024-byte boundary of the shared window, wherever the CTA's dynamic region happens to begin
  // (it is not 1024-aligned when the SM is shared with CTAs of other kernels)
  unsigned char* base = tsm + ((1024u - (smem_u32(tsm) & 1023u)) & 1023u);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  // warp -> 32 x 16 sub-tile.  The column group rotates with the tile row so that the warps of a
  // ragged last column tile that own no valid column (they skip the k-loop: "live") idle a
  // different SM sub-partition in every CTA -- warp w issues on sub-partition w % 4, and with a
  // fixed mapping sub-partitions 0 / 1 would stay the bottleneck (M0 = 152: 3 tiles of 64)
  const int wm = (warp / NWC) * 32, wn = ((warp + blockIdx.y + blockIdx.z) % NWC) * 16;
  const int m0 = blockIdx.y * TM, n0 = p.ncol0 + blockIdx.x * TNW, bz = blockIdx.z;
  const int nk = p.k / TK;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NTH / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int s, int kt) {  // elected thread
    unsigned char* st = base + (size_t)s * SB;
    mbar_arrive_expect_tx(&full[s], SB);
    if (!CONJT) {
      tma_load_3d(st, &map_are, p.acol + kt * TK, p.arow + m0, bz, &full[s]);
      tma_load_3d(st + A_BYTES, &map_aim, p.acol + kt * TK, p.arow + m0, bz, &full[s]);
    } else {  // A(r, k) = conj(M[arow + k][acol + r])
      tma_load_3d(st, &map_are, p.acol + m0, p.arow + kt * TK, bz, &full[s]);
      tma_load_3d(st + A_BYTES, &map_aim, p.acol + m0, p.arow + kt * TK, bz, &full[s]);
    }
#pragma unroll
    for (int j = 0; j < NWC; ++j) {
      tma_load_3d(st + 2 * A_BYTES + j * (TK * 128), &map_bre, p.bcol + n0 + 16 * j, p.brow + kt * TK, bz, &full[s]);
      tma_load_3d(st + 2 * A_BYTES + BB + j * (TK * 128), &map_bim, p.bcol + n0 + 16 * j, p.brow + kt * TK, bz,
                  &full[s]);
    }
  };
  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < TST && s < nk; ++s) issue(s, s);
  }
  const bool live = n0 + wn < p.n;  // warp-uniform
  double accr[4][2][2], acci[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) accr[a][b][0] = accr[a][b][1] = acci[a][b][0] = acci[a][b][1] = 0.0;
  // swizzled byte offsets that do not depend on the k-step
  // A(row, k): row * 128 + ((k >> 1) ^ (row & 7)) * 16 + (k & 1) * 8
  // B(k, n):   (n >> 4) * 2048 + k * 128 + ((((n & 15) >> 1)) ^ (k & 7)) * 16 + (n & 1) * 8
  int stage = 0;
  unsigned phase = 0;
  for (int kt = 0; kt < nk; ++kt) {
    mbar_wait_parity(&full[stage], phase);
    const unsigned char* st = base + (size_t)stage * SB;
    if (live) {
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int kk = (s4 >> 1) * 8 + (s4 & 1) * 2 + (q & 1) + 4 * (q >> 1);
        double x[4], y[4], z[4], br[2], bi[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int n = wn + t * 8 + g;
          const int off = (n >> 4) * 2048 + kk * 128 + ((((n & 15) >> 1) ^ (kk & 7)) << 4) + ((n & 1) << 3);
          br[t] = *reinterpret_cast<const double*>(st + 2 * A_BYTES + off);
          bi[t] = *reinterpret_cast<const double*>(st + 2 * A_BYTES + BB + off);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int r = wm + t * 8 + g;
          const int off = CONJT ? kk * (TM * 8) + r * 8 : r * 128 + (((kk >> 1) ^ (r & 7)) << 4) + ((kk & 1) << 3);
          const double ar = *reinterpret_cast<const double*>(st + off);
          const double ai = *reinterpret_cast<const double*>(st + A_BYTES + off);
          const double nar = __longlong_as_double(__double_as_longlong(ar) ^ 0x8000000000000000ull);
          const double nai = __longlong_as_double(__double_as_longlong(ai) ^ 0x8000000000000000ull);
          // -(A B): re += (-ar) br + ai bi, im += (-ar) bi + (-ai) br; conj(A) flips the sign of ai
          x[t] = nar;
          y[t] = CONJT ? nai : ai;
          z[t] = CONJT ? ai : nai;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            dmma(accr[a][b][0], accr[a][b][1], x[a], br[b]);
            dmma(acci[a][b][0], acci[a][b][1], x[a], bi[b]);
          }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            dmma(accr[a][b][0], accr[a][b][1], y[a], bi[b]);
            dmma(acci[a][b][0], acci[a][b][1], z[a], br[b]);
          }
      }
    }
    // This warp is done with the stage; the elected thread refills it once all 8 warps are.
    // The refill is an ASYNC-proxy write (bulk tensor copy) to memory this warp has just read
    // through the generic proxy (LDS): the release needs a proxy fence, and it must not overtake
    // the loads.  Without either, ptxas placed the arrive right after the last LDS was ISSUED (the
    // DMMAs that consume the fragments followed it), and under bank-conflict replays with two CTAs
    // per SM the refill of a B box -- an L2 hit -- landed before a late warp had read the old box:
    // one wrong 16-column sub-tile in about one sweep pass in three for the transposed form
    // (tools/soak_blocked_sweeps.py).  Two measures, each clean on its own in 71 repeat passes:
    //  * fence.proxy.async orders the generic-proxy reads before later async-proxy accesses;
    //  * lane 0 first stores a word that depends on every accumulator, so the arrive cannot
    //    issue before the stage's DMMAs -- hence all their operand loads -- have completed.
    unsigned dep = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) dep ^= (unsigned)__double2hiint(accr[a][b][0]) ^ (unsigned)__double2hiint(acci[a][b][0]);
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if (lane == 0) {
      sink[warp] = dep;
      mbar_arrive(&empty[stage]);
    }
    if (tid == 0 && kt + TST < nk) {
      mbar_wait_parity(&empty[stage], phase);
      issue(stage, kt + TST);
    }
    if (++stage == TST) {
      stage = 0;
      phase ^= 1;
    }
  }
  // C += product (one rounding per element), half a tile's loads in flight at a time
  double* cre = p.cre + bz * p.sc;
  double* cim = p.cim + bz * p.sc;
#pragma unroll
  for (int a0 = 0; a0 < 4; a0 += 2) {
    double2 lr[2][2], li[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int i = m0 + wm + (a0 + a) * 8 + g, j = n0 + wn + b * 8 + 2 * q;
        const long long c = (long long)i * p.ldc + j;
        lr[a][b] = li[a][b] = make_double2(0.0, 0.0);
        if (i < p.m && j + 1 < p.n) {
          lr[a][b] = *reinterpret_cast<const double2*>(cre + c);
          li[a][b] = *reinterpret_cast<const double2*>(cim + c);
        } else if (i < p.m && j < p.n) {
          lr[a][b].x = cre[c];
          li[a][b].x = cim[c];
        }
      }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int i = m0 + wm + (a0 + a) * 8 + g, j = n0 + wn + b * 8 + 2 * q;
        const long long c = (long long)i * p.ldc + j;
        const double2 orr = make_double2(lr[a][b].x + accr[a0 + a][b][0], lr[a][b].y + accr[a0 + a][b][1]);
        const double2 oi = make_double2(li[a][b].x + acci[a0 + a][b][0], li[a][b].y + acci[a0 + a][b][1]);
        if (i < p.m && j + 1 < p.n) {
          *reinterpret_cast<double2*>(cre + c) = orr;
          *reinterpret_cast<double2*>(cim + c) = oi;
        } else if (i < p.m && j < p.n) {
          cre[c] = orr.x;
          cim[c] = oi.x;
        }
      }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const double* base, int rows, int cols, long long ld, long long batch_stride, int count,
              int box_rows, int box_cols = 16) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)count};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)batch_stride * 8};
  const cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};  // 16 columns = one 128-byte swizzle row
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool lu_tma_maps_make_rect(LuTmaMaps* t, const double* re, const double* im, int rows, int cols, long long ld,
                           long long stride, int count) {
  t->ok = false;
  if (rows < 1 || cols < 1 || (ld & 1) || (stride & 1) || ((uintptr_t)re & 15) || ((uintptr_t)im & 15)) return false;
  if (count > 1 && stride <= 0) return false;
  static_assert(sizeof(t->m) >= 6 * sizeof(CUtensorMap), "LuTmaMaps storage");
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(t->m);
  const long long bs = count > 1 ? stride : (long long)rows * ld;  // any valid stride for a single item
  t->ok = make_map(m + 0, re, rows, cols, ld, bs, count, TM) && make_map(m + 1, im, rows, cols, ld, bs, count, TM) &&
          make_map(m + 2, re, rows, cols, ld, bs, count, TK) && make_map(m + 3, im, rows, cols, ld, bs, count, TK) &&
          make_map(m + 4, re, rows, cols, ld, bs, count, TK, TM) && make_map(m + 5, im, rows, cols, ld, bs, count, TK, TM);
  return t->ok;
}

bool lu_tma_maps_make(LuTmaMaps* t, const double* re, const double* im, int n, long long ld, long long slu, int count) {
  if (n < 64) {
    t->ok = false;
    return false;
  }
  return lu_tma_maps_make_rect(t, re, im, n, n, ld, slu, count);
}

constexpr size_t SMEM64 = (size_t)TST * STAGE_BYTES + 1024;                       // + slack to align the tiles to 1024 bytes
constexpr size_t SMEM32 = (size_t)TST * (2 * A_BYTES + 2 * TK * 32 * 8) + 1024;  // the 32-column form

static void tma_kernel_config() {
  static DevOnce cfg;
  if (cfg.first()) {
    cudaFuncSetAttribute(zgemm_tma_kernel<false, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM64);
    cudaFuncSetAttribute(zgemm_tma_kernel<true, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM64);
    cudaFuncSetAttribute(zgemm_tma_kernel<false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM32);
    cudaFuncSetAttribute(zgemm_tma_kernel<true, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM32);
  }
}

cudaError_t zgemm_tma_sub(const LuTmaMaps& ta, const LuTmaMaps& tb, double* cre, double* cim, long long ldc,
                          long long sc, int count, int m, int n, int k, int arow, int acol, int brow, int bcol,
                          cudaStream_t st, bool conjt) {
  if (m <= 0 || n <= 0 || k <= 0) return cudaSuccess;
  if (!ta.ok || !tb.ok || (ldc & 1) || ((uintptr_t)cre & 15) || ((uintptr_t)cim & 15)) return cudaErrorNotSupported;
  const CUtensorMap* mp = reinterpret_cast<const CUtensorMap*>(ta.m);
  const CUtensorMap* mq = reinterpret_cast<const CUtensorMap*>(tb.m);
  TmaArgs a{};
  a.m = m; a.n = n; a.k = ceil_div(k, TK) * TK;  // a K tail reads zero-filled entries past the tensors' edge
  a.arow = arow; a.acol = acol; a.brow = brow; a.bcol = bcol;
  a.cre = cre; a.cim = cim; a.ldc = ldc; a.sc = sc;
  tma_kernel_config();
  // 64-column tiles, and a ragged tail of at most 32 columns on the 32-column form
  const int rem = n % TN, tail = (rem > 0 && rem <= 32) ? rem : 0;
  const int wide = (n - tail + TN - 1) / TN;
  if (wide > 0) {
    const dim3 grid(wide, ceil_div(m, TM), count);
    a.ncol0 = 0;
    if (conjt)
      zgemm_tma_kernel<true, 64><<<grid, 256, SMEM64, st>>>(mp[4], mp[5], mq[2], mq[3], a);
    else
      zgemm_tma_kernel<false, 64><<<grid, 256, SMEM64, st>>>(mp[0], mp[1], mq[2], mq[3], a);
    count_launch();
  }
  if (tail > 0) {
    const dim3 grid(1, ceil_div(m, TM), count);
    a.ncol0 = n - tail;
    if (conjt)
      zgemm_tma_kernel<true, 32><<<grid, 128, SMEM32, st>>>(mp[4], mp[5], mq[2], mq[3], a);
    else
      zgemm_tma_kernel<false, 32><<<grid, 128, SMEM32, st>>>(mp[0], mp[1], mq[2], mq[3], a);
    count_launch();
  }
  return cudaGetLastError();
}

// C(m x n at M[crow][ccol]) -= A(m x k at M[arow][acol]) * B(k x n at M[brow][bcol]) for every batch item
cudaError_t lu_trailing_tma(const LuTmaMaps& t, double* re, double* im, long long ld, long long slu, int count, int m,
                            int n, int k, int arow, int acol, int brow, int bcol, int crow, int ccol, cudaStream_t st) {
  if (m <= 0 || n <= 0 || k <= 0) return cudaSuccess;
  if (!t.ok || (k % TK) != 0 || (ccol & 1)) return cudaErrorNotSupported;
  const CUtensorMap* mp = reinterpret_cast<const CUtensorMap*>(t.m);
  TmaArgs a{};
  a.m = m; a.n = n; a.k = k; a.arow = arow; a.acol = acol; a.brow = brow; a.bcol = bcol;
  a.cre = re + (long long)crow * ld + ccol;
  a.cim = im + (long long)crow * ld + ccol;
  a.ldc = ld; a.sc = slu;
  a.ncol0 = 0;
  tma_kernel_config();
  zgemm_tma_kernel<false, 64><<<dim3(ceil_div(n, TN), ceil_div(m, TM), count), 256, SMEM64, st>>>(mp[0], mp[1], mp[2], mp[3], a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace fb
