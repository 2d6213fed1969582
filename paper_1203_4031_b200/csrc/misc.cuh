#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

cudaError_t splitmix_launch(unsigned long long seed, long long off_re, long long off_im, int n, int m,
                            double* re, double* im, long long ld, cudaStream_t st);
cudaError_t accumulate_launch(int mode, int n, int m, const double* xr, const double* xi,
                              long long ldx, double* qr, double* qi, long long ldq, double h,
                              double cr, double ci, cudaStream_t st);
// one contour pass's quadrature terms (<= kMaxAccTerms), applied in order
constexpr int kMaxAccTerms = 64;
struct AccTerms {
  int count;
  int mode[kMaxAccTerms];
  double h[kMaxAccTerms], cr[kMaxAccTerms], ci[kMaxAccTerms];
  const double* xr[kMaxAccTerms];
  const double* xi[kMaxAccTerms];
};
cudaError_t accumulate_terms_launch(const AccTerms& t, int n, int m, long long ldx, double* qr, double* qi,
                                    long long ldq, cudaStream_t st);
cudaError_t symmetrize_launch(int m, double* re, double* im, long long ld, cudaStream_t st);
size_t residual_scratch_bytes(int n, int m);
cudaError_t residual_launch(int n, int m, const double* axr, const double* axi, const double* bxr,
                            const double* bxi, long long ld, const double* lam, double scale,
                            double* res, double* scratch, cudaStream_t st);
cudaError_t residual_sums_launch(int n, int m, const double* axr, const double* axi, const double* bxr,
                                 const double* bxi, long long ld, const double* lam, double scale,
                                 double* sums, double* scratch, cudaStream_t st);
cudaError_t pack_launch(int n, int m, const double* z, long long ldz, double* re, double* im,
                        long long ldp, int to_planar, cudaStream_t st);

// reduced eigensolver (reduced.cu)
size_t reduced_scratch_bytes(int m);
cudaError_t chol_check_launch(int m, const double* bre, const double* bim, long long ld, int* fail,
                              double* scratch, cudaStream_t st);
cudaError_t reduced_eig_launch(int m, const double* are, const double* aim, const double* bre,
                               const double* bim, long long ld, double* eps, double* phre,
                               double* phim, long long ldphi, int* status, double* scratch,
                               cudaStream_t st);
// cluster (DSMEM-resident) variant for M0 <= 256 (reduced_cluster.cu)
bool reduced_cluster_ok(int m, bool cplx);
size_t reduced_cluster_scratch_bytes(int m);
cudaError_t reduced_cluster_launch(int m, const double* are, const double* aim, const double* bre,
                                   const double* bim, long long ld, double* eps, double* phre, double* phim,
                                   long long ldphi, int* status, double* scratch, int check_only,
                                   cudaStream_t st);

}  // namespace fb
