// Variant harness for the thread-per-matrix batch kernels (C2a / C2b shapes).
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_2510_03421_b200/csrc/batch.cuh"
using namespace permb200;
// experiment: no shared-memory staging, each thread reads its matrix through L1
template <typename T, int N, int TPB>
__global__ void __launch_bounds__(TPB) glynn_l1_kernel(const T* __restrict__ a, T* __restrict__ out, int64_t nb) {
  const int64_t i = (int64_t)blockIdx.x * TPB + threadIdx.x;
  if (i < nb) out[i] = Num<T>::scale(1.0 / (double)(1 << (N - 1)), batch_glynn_one<T, N>(a + i * N * N));
}
template <typename K>
float timeit(K launch, int reps) {
  launch();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}
int main() {
  const int64_t B = 1000000;
  std::vector<double> h(B * 64);
  std::mt19937_64 g(1); std::normal_distribution<double> nd(0, 0.35);
  for (auto& x : h) x = nd(g);
  double *a, *out; cudaMalloc(&a, h.size() * 8); cudaMalloc(&out, B * 8);
  cudaMemcpy(a, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  {
    constexpr int STRIDE = 64 | 1;
    size_t smem = (size_t)kBatchThreads * STRIDE * 8;
    cudaFuncSetAttribute(batch_glynn_kernel<double, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float ms = timeit([&] { batch_glynn_kernel<double, 8><<<(B + kBatchThreads - 1) / kBatchThreads, kBatchThreads, smem>>>(a, out, B); }, 10);
    printf("threads=%d glynn 8x8 1e6: %.4f ms  %.2f Tops  err=%s\n", kBatchThreads, ms, B * 2048.0 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  {
    float ms32 = timeit([&] { glynn_l1_kernel<double, 8, 32><<<(B + 31) / 32, 32>>>(a, out, B); }, 10);
    float ms64 = timeit([&] { glynn_l1_kernel<double, 8, 64><<<(B + 63) / 64, 64>>>(a, out, B); }, 10);
    float ms128 = timeit([&] { glynn_l1_kernel<double, 8, 128><<<(B + 127) / 128, 128>>>(a, out, B); }, 10);
    printf("L1-direct glynn 8x8 1e6: tpb32 %.4f ms, tpb64 %.4f ms, tpb128 %.4f ms err=%s\n", ms32, ms64, ms128,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    constexpr int STRIDE = 40 | 1;
    size_t smem = (size_t)kBatchThreads * STRIDE * 8;
    cudaFuncSetAttribute(batch_ryser_kernel<double, 4, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float ms = timeit([&] { batch_ryser_kernel<double, 4, 10><<<(B + kBatchThreads - 1) / kBatchThreads, kBatchThreads, smem>>>(a, out, B); }, 10);
    printf("threads=%d ryser 4x10 1e6: %.4f ms  err=%s\n", kBatchThreads, ms, cudaGetErrorString(cudaGetLastError()));
  }
  {
    constexpr int STRIDE = 40 | 1;
    size_t smem = (size_t)kBatchThreads * STRIDE * 8;
    cudaFuncSetAttribute(batch_combdp_kernel<double, 4, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float ms = timeit([&] { batch_combdp_kernel<double, 4, 10><<<(B + kBatchThreads - 1) / kBatchThreads, kBatchThreads, smem>>>(a, out, B); }, 10);
    printf("threads=%d combdp 4x10 1e6: %.4f ms  %.1f GB/s err=%s\n", kBatchThreads, ms, B * 320.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
