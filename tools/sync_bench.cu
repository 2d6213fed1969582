// Barrier latency microbenchmark on B200: cluster.sync (+DSMEM read), grid.sync, __syncthreads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cluster(int iters, double* out) {
  __shared__ double buf[64];
  auto cl = cg::this_cluster();
  buf[threadIdx.x & 63] = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    cl.sync();
    if (threadIdx.x < 32) {
      const double* r = cl.map_shared_rank(buf, (cl.block_rank() + 1) % cl.num_blocks());
      acc += r[threadIdx.x];
    }
  }
  cl.sync();
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_cluster_only(int iters, double* out) {
  auto cl = cg::this_cluster();
  for (int i = 0; i < iters; ++i) cl.sync();
}
__global__ void k_grid(int iters, double* out) {
  auto g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}
__global__ void k_block(int iters, double* out) {
  __shared__ double s[256];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    s[threadIdx.x] = i;
    __syncthreads();
    acc += s[(threadIdx.x + 1) & 255];
    __syncthreads();
  }
  if (acc == 1.0) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  float ms;
  for (int cs : {2, 4, 8, 16}) {
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_cluster_only, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int which = 0; which < 2; ++which) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256); cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, which ? k_cluster_only : k_cluster, 10, out);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, which ? k_cluster_only : k_cluster, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("cluster=%2d %s: %.3f us/iter (%s)\n", cs, which ? "sync only " : "sync+dsmem", ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int g : {16, 32, 148, 296}) {
    void* args[] = {(void*)&iters, (void*)&out};
    int it2 = 10;
    void* args2[] = {(void*)&it2, (void*)&out};
    cudaLaunchCooperativeKernel((void*)k_grid, dim3(g), dim3(128), args2, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_grid, dim3(g), dim3(128), args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid=%3d: %.3f us/iter (%s)\n", g, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  k_block<<<1, 256>>>(10, out);
  cudaEventRecord(e0);
  k_block<<<1, 256>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("syncthreads x2: %.3f us/iter\n", ms * 1e3 / iters);
  return 0;
}
