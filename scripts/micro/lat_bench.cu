// Micro-benchmark: latency of block 0 reading data written by another SM in
// the previous grid-barrier phase, vs data written by itself, vs old data,
// at several distances from a hot line (TLB reach).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_lat(double* buf, long stride_elems, int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long acc[6] = {0, 0, 0, 0, 0, 0};
  double sink = 0;
  for (int it = 0; it < iters; ++it) {
    // phase 1: block 5 writes buf[it % 64 * 8 + 1], block 0 writes buf[2]
    if (threadIdx.x == 0 && blockIdx.x == 5) buf[(it % 64) * 16 + 1] = it;
    if (threadIdx.x == 0 && blockIdx.x == 0) buf[2] = it;
    g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      unsigned long long t0 = clock64();
      double a = *(volatile double*)&buf[(it % 64) * 16 + 1];  // written by another SM
      sink += a;
      unsigned long long t1 = clock64();
      double b = *(volatile double*)&buf[2];  // written by me
      sink += b;
      unsigned long long t2 = clock64();
      double c = *(volatile double*)&buf[4096 + (it % 64) * 16];  // never written, near
      sink += c;
      unsigned long long t3 = clock64();
      double d = *(volatile double*)&buf[stride_elems + (it % 64) * 16];  // far (other page)
      sink += d;
      unsigned long long t4 = clock64();
      double e = *(volatile double*)&buf[3 * stride_elems + (it % 64) * 16];  // farther
      sink += e;
      unsigned long long t5 = clock64();
      double f = *(volatile double*)&buf[(it % 64) * 16 + 1];  // again (now cached?)
      sink += f;
      unsigned long long t6 = clock64();
      acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3; acc[4] += t5 - t4; acc[5] += t6 - t5;
    }
    g.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (int k = 0; k < 6; ++k) out[k] = acc[k] / iters;
    out[6] = (unsigned long long)sink;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double* buf;
  size_t bytes = (size_t)8 << 30;  // 8 GiB
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  unsigned long long* out;
  cudaMallocManaged(&out, 64);
  for (long stride : {1L << 18, 1L << 24, 1L << 28}) {  // 2 MiB, 128 MiB, 2 GiB (in doubles x8 bytes)
    int iters = 2000;
    void* args[] = {&buf, &stride, &iters, &out};
    cudaLaunchCooperativeKernel((void*)k_lat, 148, 256, args, 0, 0);
    cudaDeviceSynchronize();
    printf("stride=%ld doubles: other-SM-written=%llu self-written=%llu near-untouched=%llu far=%llu farther=%llu reread=%llu cycles (%s)\n",
           stride, out[0], out[1], out[2], out[3], out[4], out[5], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
