#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

size_t zgetrf_scratch_bytes(int n);
size_t dinv_doubles(int n);
const int* factor_perm(const double* dinv, int n);
cudaError_t shift_launch(int n, double zr, double zi, const double* are, const double* aim,
                         long long lda, const double* bre, const double* bim, long long ldb,
                         double* sre, double* sim, long long lds, cudaStream_t st);
cudaError_t permute_rows_launch(int n, int m, const int* perm, int gather, const double* ir,
                                const double* ii, long long ldi, double* orr, double* oi,
                                long long ldo, cudaStream_t st);
struct LuStreams {
  cudaStream_t side;   // high-priority stream for the look-ahead panels (nullptr: none)
  cudaEvent_t ev_s;    // recorded on the main stream
  cudaEvent_t ev_p;    // recorded on the side stream
};
cudaError_t zgetrf(int n, double* re, double* im, long long ld, int* piv, int* info, double* dinv,
                   char* scratch, cudaStream_t st, const LuStreams* ls);
cudaError_t zgetrs(int n, int nrhs, const double* re, const double* im, long long ld, const int* piv,
                   const double* dinv, int adjoint, double* xr, double* xi, long long ldx, double* tmp,
                   cudaStream_t st);

}  // namespace fb
