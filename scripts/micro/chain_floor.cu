// Latency floor of one deep-dive iteration's exchange pattern on this GPU:
// every block publishes a partial (10 doubles), a grid barrier, every block
// reads all G partials back (one L2 round trip) and reduces them (warp
// shuffles + shared memory), a block barrier -- the minimum a k_chain
// iteration must pay whatever its arithmetic (roofline of the
// latency-bound headline).  Also: the same with a 16-CTA cluster and DSMEM.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 1) k_floor(int iters, double* part, double* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ double s_w[8];
  double acc = 0.0;
  for (int k = 0; k < iters; ++k) {
    double* P = part + (size_t)(k & 1) * gridDim.x * 16;
    if (threadIdx.x < 10) P[blockIdx.x * 16 + threadIdx.x] = acc + threadIdx.x + k;
    g.sync();
    double v = 0.0;
    if (threadIdx.x < gridDim.x)
      for (int q = 0; q < 5; ++q) v += __ldcg(&P[threadIdx.x * 16 + q]);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w) v += s_w[w];
      s_w[0] = v;
    }
    __syncthreads();
    acc = s_w[0] * 1e-30;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = acc;
}

template <int CS>
__global__ void __launch_bounds__(256, 1) k_floor_cl(int iters, double* sink) {
  cg::cluster_group c = cg::this_cluster();
  __shared__ double s_part[2][16];
  __shared__ double s_w[8];
  double acc = 0.0;
  for (int k = 0; k < iters; ++k) {
    if (threadIdx.x < 10) s_part[k & 1][threadIdx.x] = acc + threadIdx.x + k;
    c.sync();
    double v = 0.0;
    if (threadIdx.x < CS)
      for (int q = 0; q < 5; ++q) v += c.map_shared_rank(&s_part[k & 1][0], threadIdx.x)[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w) v += s_w[w];
      s_w[0] = v;
    }
    __syncthreads();
    acc = s_w[0] * 1e-30;
  }
  c.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *part, *sink;
  cudaMalloc(&part, 2 * 16 * 1024 * sizeof(double));
  cudaMalloc(&sink, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 20000;
  printf("{\"sms\": %d", sms);
  for (int G : {sms, 64, 32, 16}) {
    void* args[] = {&iters, &part, &sink};
    cudaLaunchCooperativeKernel((void*)k_floor, G, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_floor, G, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf(", \"grid_%d_us_per_iter\": %.3f", G, ms * 1e3 / iters);
  }
  {
    cudaFuncSetAttribute((const void*)k_floor_cl<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_floor_cl<16>, iters, sink);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k_floor_cl<16>, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf(", \"cluster16_dsmem_us_per_iter\": %.3f", ms * 1e3 / iters);
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
