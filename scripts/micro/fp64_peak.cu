// fp64_peak.cu -- measured FP64 throughput of one B200 for the roofline
// denominator (bench.py "roofline.peak" when bound = "fp64").  Every kernel
// keeps 8 independent dependency chains per thread (enough to cover the FP64
// pipe latency), 148 x 8 blocks of 256 threads, and reports instructions per
// second; DFMA counts 2 flops, DADD / DMUL 1.  The directed-rounding variants
// (.RD / .RP) are the instructions the interval kernels issue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8, ITERS = 4096;

enum Op { FMA_RN, ADD_RN, ADD_RD, ADD_RU, MUL_RD, MUL_RU, ADDRDRU };

template <int OP>
__global__ void __launch_bounds__(256) k(const double* in, double* out) {
  double a[CH];
  const double b = in[0], c = in[1];
#pragma unroll
  for (int j = 0; j < CH; ++j) a[j] = in[2 + j] + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      if (OP == FMA_RN) a[j] = fma(a[j], b, c);
      if (OP == ADD_RN) a[j] = __dadd_rn(a[j], b);
      if (OP == ADD_RD) a[j] = __dadd_rd(a[j], b);
      if (OP == ADD_RU) a[j] = __dadd_ru(a[j], b);
      if (OP == MUL_RD) a[j] = __dmul_rd(a[j], b);
      if (OP == MUL_RU) a[j] = __dmul_ru(a[j], b);
      if (OP == ADDRDRU) a[j] = (j & 1) ? __dadd_ru(a[j], b) : __dadd_rd(a[j], c);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += a[j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int OP>
double run(const double* in, double* out, int blocks, double* ms_out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<OP><<<blocks, 256>>>(in, out);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k<OP><<<blocks, 256>>>(in, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  *ms_out = best;
  return (double)blocks * 256 * CH * ITERS / (best * 1e-3);  // instructions / s
}

int main() {
  double h[16] = {1.0000000001, 1e-300, 1, 2, 3, 4, 5, 6, 7, 8};
  double *in, *out;
  cudaMalloc(&in, sizeof h);
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  int sms = 148, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8;
  const char* names[] = {"dfma_rn", "dadd_rn", "dadd_rd", "dadd_ru", "dmul_rd", "dmul_ru", "dadd_rd_ru_mix"};
  double ips[7], ms[7];
  ips[0] = run<FMA_RN>(in, out, blocks, &ms[0]);
  ips[1] = run<ADD_RN>(in, out, blocks, &ms[1]);
  ips[2] = run<ADD_RD>(in, out, blocks, &ms[2]);
  ips[3] = run<ADD_RU>(in, out, blocks, &ms[3]);
  ips[4] = run<MUL_RD>(in, out, blocks, &ms[4]);
  ips[5] = run<MUL_RU>(in, out, blocks, &ms[5]);
  ips[6] = run<ADDRDRU>(in, out, blocks, &ms[6]);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"blocks\": %d, \"threads\": 256, \"chains\": %d, \"iters\": %d",
         sms, clk, blocks, CH, ITERS);
  for (int i = 0; i < 7; ++i)
    printf(", \"%s\": {\"ginstr_per_s\": %.1f, \"per_sm_per_clk_at_1965\": %.2f, \"ms\": %.4f}", names[i],
           ips[i] / 1e9, ips[i] / sms / 1.965e9, ms[i]);
  printf(", \"fp64_tflops_dfma\": %.3f, \"fp64_tops_dadd_directed\": %.3f}\n", 2 * ips[0] / 1e12, ips[6] / 1e12);
  return cudaGetLastError() != cudaSuccess;
}
