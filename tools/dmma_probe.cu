// Does the FP64 tensor path (mma.sync m8n8k4 f64, "DMMA") run beside the
// FP64 vector pipe (DFMA)?  Times DFMA-only, DMMA-only and an interleaved
// kernel; if mixed ~ max(alone) the pipes are separate and the Gray walk's
// state updates could be offloaded to DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <bool DO_FMA, bool DO_MMA>
__global__ void probe(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0, c7 = 0;
  double ma = a * threadIdx.x, mb = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (DO_FMA) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      }
      if (DO_MMA && (u & 1) == 0) {
        dmma(c0, c1, ma, mb); dmma(c2, c3, ma, mb); dmma(c4, c5, ma, mb); dmma(c6, c7, ma, mb);
      }
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
  if (s == 12345.678) out[0] = s;
}

template <bool F, bool M>
float run(int blocks, int tpb, int iters, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) probe<F, M><<<blocks, tpb>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) probe<F, M><<<blocks, tpb>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 8);
  int iters = 2048, tpb = 256, blocks = p.multiProcessorCount * 8;
  double thr = (double)blocks * tpb;
  float tf = run<true, false>(blocks, tpb, iters, out);
  float tm = run<false, true>(blocks, tpb, iters, out);
  float tb = run<true, true>(blocks, tpb, iters, out);
  double dfma = thr * iters * 128, mmas = thr / 32 * iters * 32;  // 8 per iter-unroll -> 4*8=32 per iter
  printf("dfma-only  %.3f ms  %.4e DFMA/s\n", tf, dfma / (tf * 1e-3));
  printf("dmma-only  %.3f ms  %.4e DMMA/s = %.4e FP64 MAC/s (256 MAC each)\n", tm, mmas / (tm * 1e-3),
         256 * mmas / (tm * 1e-3));
  printf("both       %.3f ms  (sum of alone %.3f, max %.3f)\n", tb, tf + tm, tf > tm ? tf : tm);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
