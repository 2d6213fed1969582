#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

size_t gmat_doubles(int n);
cudaError_t gmat_launch(int n, const double* lre, const double* lim, long long ld, const double* dinv,
                        double* gmat, cudaStream_t st);
cudaError_t sweep_launch(int variant, int n, int nrhs, const double* lre, const double* lim, long long ld,
                         const double* dinv, const double* gmat, double* xre, double* xim, long long ldx,
                         cudaStream_t st);

}  // namespace fb
