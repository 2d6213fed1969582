#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

size_t gmat_doubles(int n);
cudaError_t gmat_launch(int n, int count, const double* lre, const double* lim, long long ld, long long slu,
                        const double* dinv, long long sdinv, double* gmat, cudaStream_t st);
cudaError_t sweep_launch(int variant, int n, int nrhs, int count, const double* lre, const double* lim,
                         long long ld, long long slu, const double* dinv, const double* gmat, long long sdinv,
                         double* xre, double* xim, long long ldx, long long sx, cudaStream_t st);

}  // namespace fb
