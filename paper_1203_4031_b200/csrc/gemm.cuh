#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

struct Opnd {
  const double* re;
  const double* im;  // nullptr: imaginary part is zero (real operand)
  long long s0, s1;  // op(X)(r, c) at re[r*s0 + c*s1]
  int conj;          // conjugate the imaginary part
};

struct GemmParams {
  int m, n, k;
  Opnd a, b;
  double* cre;
  double* cim;
  long long cs0, cs1;
  double alpha_re, alpha_im, beta_re, beta_im;
  double* ws;  // split-K workspace (gemm_workspace_bytes)
  int splits;
  int kchunk;
  int batch = 1;                  // strided batch: item b uses pointers + b * bs{a,b,c}
  long long bsa = 0, bsb = 0, bsc = 0;
};

// Row-major planar helpers: X is rows x cols with leading dimension ld.
inline Opnd op_n(const double* re, const double* im, long long ld) { return {re, im, ld, 1, 0}; }
inline Opnd op_t(const double* re, const double* im, long long ld) { return {re, im, 1, ld, 0}; }
inline Opnd op_c(const double* re, const double* im, long long ld) { return {re, im, 1, ld, 1}; }

cudaError_t gemm_launch(int cplx, GemmParams p, cudaStream_t st);
size_t gemm_workspace_bytes(int cplx, int m, int n, int splits);
int gemm_pick_splits(int m, int n, int k);

// Convenience: C = alpha op(A) op(B) + beta C without split-K.
inline cudaError_t gemm(int cplx, int m, int n, int k, Opnd a, Opnd b, double* cre, double* cim,
                        long long ldc, double ar, double ai, double br, double bi, cudaStream_t st,
                        double* ws = nullptr, int splits = 1, int batch = 1, long long bsa = 0,
                        long long bsb = 0, long long bsc = 0) {
  GemmParams p;
  p.batch = batch; p.bsa = bsa; p.bsb = bsb; p.bsc = bsc;
  p.m = m; p.n = n; p.k = k; p.a = a; p.b = b;
  p.cre = cre; p.cim = cim; p.cs0 = ldc; p.cs1 = 1;
  p.alpha_re = ar; p.alpha_im = ai; p.beta_re = br; p.beta_im = bi;
  p.ws = ws; p.splits = ws ? splits : 1; p.kchunk = 0;
  return gemm_launch(cplx, p, st);
}

// TMA-fed trailing update of the blocked LU (gemm_tma.cu): tensor maps over the
// strided batch of factor matrices, made once per factorization
struct LuTmaMaps {
  alignas(64) unsigned char m[6 * 128];  // 6 CUtensorMap: (re, im) x (A box, B box, transposed-A box)
  bool ok = false;
};
bool lu_tma_maps_make(LuTmaMaps* t, const double* re, const double* im, int n, long long ld, long long slu, int count);
// the same four maps over a batch of rows x cols planar blocks (the sweeps' right-hand sides)
bool lu_tma_maps_make_rect(LuTmaMaps* t, const double* re, const double* im, int rows, int cols, long long ld,
                           long long stride, int count);
// C(m x n) -= A(m x k at A-tensor [arow][acol]) * B(k x n at B-tensor [brow][bcol]) for every batch item;
// A tiles come from ta, B tiles from tb; k is a multiple of 16 or ends at the tensors' edge.
// conjt: A(r, kk) = conj(A-tensor[arow + kk][acol + r]) instead (the adjoint sweeps' M^H).
cudaError_t zgemm_tma_sub(const LuTmaMaps& ta, const LuTmaMaps& tb, double* cre, double* cim, long long ldc,
                          long long sc, int count, int m, int n, int k, int arow, int acol, int brow, int bcol,
                          cudaStream_t st, bool conjt = false);
cudaError_t lu_trailing_tma(const LuTmaMaps& t, double* re, double* im, long long ld, long long slu, int count, int m,
                            int n, int k, int arow, int acol, int brow, int bcol, int crow, int ccol, cudaStream_t st);

}  // namespace fb
