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

// partitioned (SPIKE) band LU / solve, batched over shifts (band_spike.cu)
bool band_spike_ok(int kl);
void band_spike_set_part_target(int t);  // 0: default (4096 rows)
int band_spike_parts(int n, int kl);
size_t band_spike_aux_doubles(int n, int kl);
size_t band_spike_solve_scratch_doubles(int n, int kl, int nrhs, int count);
cudaError_t band_spike_factor(int count, int n, int kl, const double* zr, const double* zi, const double* far_,
                              const double* fai, const double* fbr, const double* fbi, long long ldb,
                              double* wr, double* wi, long long sw, int* ipiv, long long sp, double* aux,
                              long long sa, int* info, cudaStream_t st);
cudaError_t band_spike_solve(int count, int n, int kl, int nrhs, const double* wr, const double* wi, long long sw,
                             const int* ipiv, long long sp, const double* aux, long long sa, double* xr,
                             double* xi, long long ldx, long long sx, double* scratch, cudaStream_t st,
                             const double* yr = nullptr, const double* yi = nullptr, long long ldy = 0,
                             long long sy = 0);
struct AccTerms;
cudaError_t band_spike_solve_accumulate(int count, int n, int kl, int nrhs, const double* wr, const double* wi,
                                        long long sw, const int* ipiv, long long sp, const double* aux, long long sa,
                                        double* xr, double* xi, long long ldx, long long sx, double* scratch,
                                        cudaStream_t st, const double* yr, const double* yi, long long ldy,
                                        const AccTerms& terms, const int* item, double* qr, double* qi,
                                        long long ldq);

}  // namespace fb
