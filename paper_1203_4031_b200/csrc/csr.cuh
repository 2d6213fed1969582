#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

cudaError_t csr_spmm_launch(int n, int m, const long long* indptr, const long long* indices, const double* vr,
                            const double* vi, const double* xr, const double* xi, long long ldx, double* yr,
                            double* yi, long long ldy, const long long* order, cudaStream_t st);
cudaError_t gather_rows_launch(int n, int m, const long long* perm, const double* sr, const double* si,
                                long long lds, double* dr, double* di, long long ldd, cudaStream_t st);

int bicgstab_parts(int n);
size_t bicgstab_workspace_doubles(int n, int m, long long ld);
cudaError_t bicgstab_launch(int phase, int n, int m, const long long* indptr, const long long* indices,
                            const double* s_re, const double* s_im, const double* d_re, const double* d_im,
                            const double* b_re, const double* b_im, long long ldb, double* x_re, double* x_im,
                            long long ldx, double tol, int maxiter, int iters, double* work, long long ld,
                            int* istate, const long long* order, cudaStream_t st);

}  // namespace fb
