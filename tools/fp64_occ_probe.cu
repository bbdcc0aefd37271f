// FP64 pipe vs occupancy and ILP: DFMA/clk/SM with W warps per SM (one block
// per SM) and K independent chains per thread, 3 distinct register sources.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_occ_probe.cu -o tools/fp64_occ_probe_bin
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void probe(long long* t, int iters, const double* ab, double* out) {
  double x[K], a[K], b[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    x[k] = threadIdx.x + k;
    a[k] = ab[k];
    b[k] = ab[K + k];
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = fma(x[k], a[k], b[(k + u) % K]);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}
template <int K>
void run(int nsm, long long* dt, const double* ab, double* out) {
  for (int w : {2, 4, 6, 8, 12, 16, 24, 32}) {
    const int iters = 2048;
    probe<K><<<nsm, 32 * w>>>(dt, iters, ab, out);
    cudaDeviceSynchronize();
    long long ht[1];
    cudaMemcpy(ht, dt, 8, cudaMemcpyDeviceToHost);
    const double per_clk = 32.0 * w * iters * 8 * K / (double)ht[0];
    printf("K=%2d warps/SM=%2d : %.1f DFMA/clk/SM (%.0f%% of 64)\n", K, w, per_clk, per_clk / 64 * 100);
  }
}
int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* dt;
  double *ab, *out;
  cudaMalloc(&dt, 8 * 1024);
  cudaMalloc(&out, 8);
  cudaMalloc(&ab, 8 * 64);
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = (i < 32) ? 0.999 - 1e-4 * i : 1e-3 * i;
  cudaMemcpy(ab, h, sizeof h, cudaMemcpyHostToDevice);
  run<1>(nsm, dt, ab, out);
  run<2>(nsm, dt, ab, out);
  run<4>(nsm, dt, ab, out);
  run<8>(nsm, dt, ab, out);
  run<16>(nsm, dt, ab, out);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
