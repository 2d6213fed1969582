#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fb {

constexpr int PANEL_W = 32;
enum { PANEL_GRID = 0, PANEL_CLUSTER = 1 };

struct PanelArgs {
  double* re;
  double* im;
  long long ld;
  int n, c0, pw, rpc;
  int* piv;
  int* info;
  double* xrec;   // GRID mode exchange records (set by panel_launch)
  double* xrowr;  // GRID mode copy of row rj
  double* xu;     // GRID mode U rows of a finished sub-block
  double* linv;   // [2 planes][PW][PW] inverse of the unit-lower diagonal block
  double* uinv;   // [2 planes][PW][PW] inverse of the upper diagonal block
  int* list;      // [1 + 4*PW] (dst, src) row-interchange list of this panel
  // strided batch: item b = b0 + blockIdx.y offsets re/im by b*slu, piv by b*spiv,
  // linv/uinv by b*sdinv (doubles), list by 2*b*sdinv (ints), scratch by b*sxs
  long long slu, spiv, sdinv, sxs;
  int b0;
};

size_t panel_scratch_bytes();
cudaError_t panel_launch(PanelArgs a, int count, char* scratch, cudaStream_t st);
// upper diagonal-block inverses of a finished batched factorization (into dinv)
cudaError_t uinv_batched_launch(int n, int count, const double* re, const double* im, long long ld,
                                long long slu, double* dinv, long long sdinv, cudaStream_t st);

}  // namespace fb
