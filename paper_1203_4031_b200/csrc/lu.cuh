#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

constexpr int kMaxBatch = 64;  // shifts per batched call (Ne <= 48 in FEAST)

// A strided batch of LU factorizations: item b lives at (re, im) + b*slu,
// piv + b*spiv, dinv + b*sdinv, info[b].
struct LuBatch {
  int count;
  double* re;
  double* im;
  long long ld, slu;
  int* piv;
  long long spiv;
  int* info;
  double* dinv;
  long long sdinv;
};

struct LuStreams {
  cudaStream_t side;  // high-priority stream for the look-ahead panels (nullptr: none)
  cudaEvent_t ev_s;   // recorded on the main stream
  cudaEvent_t ev_p;   // recorded on the side stream
};

size_t zgetrf_scratch_bytes(int n, int count);
size_t dinv_doubles(int n);
const int* factor_perm(const double* dinv, int n);
const double* factor_gmat(const double* dinv, int n);
cudaError_t shift_launch(int n, int count, const double* zr, const double* zi, const double* are,
                         const double* aim, long long lda, const double* bre, const double* bim,
                         long long ldb, double* sre, double* sim, long long lds, long long ss, cudaStream_t st);
cudaError_t permute_rows_launch(int n, int m, int count, const int* perm, long long sperm, int gather,
                                const double* ir, const double* ii, long long ldi, long long sin_, double* orr,
                                double* oi, long long ldo, long long sout, cudaStream_t st);
cudaError_t zgetrf_batched(int n, const LuBatch& f, char* scratch, cudaStream_t st, const LuStreams* ls);
// leading dimension of zgetrs_batched's adjoint copy (even: 16-byte sweeps);
// tmp holds 2 * count * n * zgetrs_tmp_ld(nrhs) doubles
inline int zgetrs_tmp_ld(int nrhs) { return nrhs + (nrhs & 1); }
cudaError_t zgetrs_batched(int n, int nrhs, const LuBatch& f, int adjoint, const double* rr, const double* ri,
                           long long ldr, long long srhs, double* xr, double* xi, long long ldx, long long sx,
                           double* tmp, cudaStream_t st);

}  // namespace fb
