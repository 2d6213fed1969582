// Cost of alternating a 16-CTA cluster kernel (135 KB smem/CTA) with a
// many-CTA kernel of a different shared-memory footprint (the LU's
// panel / GEMM / swap sequence), vs each kernel launched back to back.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_cluster(int* p) {
  extern __shared__ double sm[];
  cg::this_cluster().sync();
  if (threadIdx.x == 0 && p) sm[0] = 1.0;
}
__global__ void k_grid(int* p, int smem_touch) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0 && p && smem_touch) sm[0] = 1.0;
}
int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(16, 1);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 135 * 1024;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int R = 200;
  for (int gsm : {0, 16, 70, 135}) {
    for (int mode = 0; mode < 3; ++mode) {  // 0 cluster only, 1 grid only, 2 alternate
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(a);
        for (int i = 0; i < R; ++i) {
          if (mode != 1) cudaLaunchKernelEx(&cfg, k_cluster, d);
          if (mode != 0) k_grid<<<592, 256, gsm * 1024>>>(d, gsm > 0);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      cudaEventElapsedTime(&ms, a, b);
      printf("grid smem %3d KB, mode %s: %7.2f us per iteration %s\n", gsm,
             mode == 0 ? "cluster only " : mode == 1 ? "grid only    " : "alternating  ", 1e3 * ms / R,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
