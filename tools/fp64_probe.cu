// Standalone FP64-pipe probe: DFMA throughput per SM per clock and the
// achieved DFMA/s, to pin the roofline denominator on the box.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
__global__ void clk_kernel(long long* t, int iters, double a, double b, double* out) {
  long long t0 = clock64();
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  long long t1 = clock64();
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("name=%s sms=%d cc=%d.%d clock_khz=%d regs/sm=%d smem/sm=%zu\n", p.name, p.multiProcessorCount, p.major, p.minor, clk, p.regsPerMultiprocessor, p.sharedMemPerMultiprocessor);
  double* out; cudaMalloc(&out, 8); long long* t; cudaMalloc(&t, 8 * 4096);
  int iters = 4096;
  for (int tpb : {256, 512, 1024}) {
    int blocks = p.multiProcessorCount * (2048 / tpb);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) dfma_kernel<<<blocks, tpb>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e0);
    int reps = 5;
    for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, tpb>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dfma = (double)blocks * tpb * iters * 16 * 8 * reps;
    printf("tpb=%d blocks=%d DFMA/s=%.4e TFLOPS(2/fma)=%.2f\n", tpb, blocks, dfma / (ms * 1e-3), 2 * dfma / (ms * 1e-3) / 1e12);
  }
  // per-SM per-clock: one block of 1024 threads per SM
  clk_kernel<<<p.multiProcessorCount, 1024>>>(t, iters, 0.999, 1e-3, out);
  long long ht[4096]; cudaMemcpy(ht, t, 8 * p.multiProcessorCount, cudaMemcpyDeviceToHost);
  double per_clk = 1024.0 * iters * 16 * 8 / (double)ht[0];
  printf("DFMA per clk per SM (1 block x 1024 thr) = %.2f (cycles=%lld)\n", per_clk, ht[0]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
