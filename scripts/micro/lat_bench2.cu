// Load latency of block 0 after a grid barrier, when the previous phase had
// every block write a slab of data (like clb / table writes), with and
// without __threadfence in the writers, and with 256 vs 32 threads.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_lat(double* buf, double* big, int iters, int mode, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long acc[4] = {0, 0, 0, 0};
  double sink = 0;
  for (int it = 0; it < iters; ++it) {
    // phase 1: every block writes 4 KB of `big` (512 doubles), block 5 writes buf[k]
    if (mode >= 1)
      for (int i = threadIdx.x; i < 512; i += blockDim.x) big[(size_t)blockIdx.x * 512 + i] = it + i;
    if (mode >= 2) __threadfence();
    if (threadIdx.x == 0 && blockIdx.x == 5) buf[(it % 64) * 16 + 1] = it;
    g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      unsigned long long t0 = clock64();
      double a = *(volatile double*)&buf[(it % 64) * 16 + 1];
      sink += a;
      unsigned long long t1 = clock64();
      double b = *(volatile double*)&big[(size_t)77 * 512 + (it % 64)];  // written by block 77
      sink += b;
      unsigned long long t2 = clock64();
      double c = *(volatile double*)&big[(size_t)0 * 512 + (it % 64)];  // written by me
      sink += c;
      unsigned long long t3 = clock64();
      double d = *(volatile double*)&buf[(it % 64) * 16 + 1];
      sink += d;
      unsigned long long t4 = clock64();
      acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3;
    }
    g.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (int k = 0; k < 4; ++k) out[k] = acc[k] / iters;
    out[4] = (unsigned long long)sink;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double *buf, *big;
  cudaMalloc(&buf, 1 << 20);
  cudaMalloc(&big, (size_t)148 * 512 * 8 * 2);
  unsigned long long* out;
  cudaMallocManaged(&out, 64);
  for (int mode = 0; mode < 3; ++mode)
    for (int tpb : {32, 256}) {
      int iters = 2000;
      void* args[] = {&buf, &big, &iters, &mode, &out};
      cudaLaunchCooperativeKernel((void*)k_lat, 148, tpb, args, 0, 0);
      cudaDeviceSynchronize();
      printf("mode=%d tpb=%d: buf(other SM)=%llu big(other SM)=%llu big(mine)=%llu reread=%llu cycles (%s)\n", mode, tpb,
             out[0], out[1], out[2], out[3], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
