#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

size_t band_fact_doubles(int n, int kl);
cudaError_t band_matvec_launch(int n, int kl, int m, const double* fbr, const double* fbi, long long ldb,
                               const double* xr, const double* xi, long long ldx, double* yr, double* yi,
                               long long ldy, cudaStream_t st);
cudaError_t band_factor_launch(int n, int kl, double zr, double zi, const double* far_, const double* fai,
                               const double* fbr, const double* fbi, long long ldb, double* wr, double* wi,
                               int* ipiv, int* info, cudaStream_t st);
cudaError_t band_solve_launch(int n, int kl, int nrhs, const double* wr, const double* wi, const int* ipiv,
                              int adjoint, double* xr, double* xi, long long ldx, cudaStream_t st);

}  // namespace fb
