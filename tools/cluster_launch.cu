// Launch cost of thread-block clusters (the panel kernel's shape): an empty
// kernel with G CTAs per cluster, 256 threads, S KB of dynamic shared memory,
// launched back to back; prints the mean time per launch.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void empty_cluster(int* p) {
  extern __shared__ double sm[];
  cg::this_cluster().sync();
  if (threadIdx.x == 0 && p) sm[0] = 1.0;
  cg::this_cluster().sync();
}
int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(empty_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(empty_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int gs[] = {1, 2, 4, 8, 16};
  int ss[] = {16, 135, 200};
  for (int G : gs)
    for (int S : ss)
      for (int items : {1, 8}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = G;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(G, items);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = S * 1024;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, empty_cluster, d);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        const int R = 200;
        for (int i = 0; i < R; ++i) cudaLaunchKernelEx(&cfg, empty_cluster, d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("cluster %2d x %d items, smem %3d KB: %7.2f us/launch %s\n", G, items, S, 1e3 * ms / R,
               e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
