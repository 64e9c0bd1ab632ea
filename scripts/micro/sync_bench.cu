// Micro-benchmark: cost of grid-wide barriers (cooperative groups) and of a
// hand-rolled barrier, vs grid size; cluster barrier for a 16-CTA cluster.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_grid(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = 1;
}
__global__ void k_mybar(int iters, unsigned* cnt) {
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = gridDim.x * (unsigned)(i + 1);
      __threadfence();
      atomicAdd(cnt, 1u);
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(cnt));
      } while (v < target);
    }
    __syncthreads();
  }
}
__global__ void __cluster_dims__(1, 1, 1) k_dummy() {}
__global__ void k_cluster(int iters, unsigned* sink) {
  cg::cluster_group c = cg::this_cluster();
  for (int i = 0; i < iters; ++i) c.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = 1;
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 2000;
  int grids[] = {1, 2, 8, 16, 32, 64, 148};
  for (int g : grids) {
    void* args[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)k_grid, g, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_grid, g, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cg grid.sync  grid=%3d : %.3f us/sync  (%s)\n", g, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    cudaMemset(sink, 0, 4);
    cudaLaunchCooperativeKernel((void*)k_mybar, g, 256, args, 0, 0);
    cudaMemset(sink, 0, 4);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_mybar, g, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("hand barrier  grid=%3d : %.3f us/sync  (%s)\n", g, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute((void*)k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cluster, iters, sink);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k_cluster, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster.sync  size=%3d : %.3f us/sync  (%s)\n", cs, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
