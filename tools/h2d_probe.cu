// Host->device paths for a 512 MB pageable batch (C2a size): pinned DMA,
// pageable->pinned memcpy with T threads, cudaHostRegister + DMA, direct
// pageable DMA.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
using clk = std::chrono::steady_clock;
static double ms_since(clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); }

int main() {
  const size_t N = 512ull << 20, C = 32ull << 20;
  char* src = (char*)malloc(N);
  memset(src, 1, N);
  char *pin, *dev;
  cudaMallocHost(&pin, N);
  cudaMalloc(&dev, N);
  memset(pin, 2, N);
  cudaStream_t s; cudaStreamCreate(&s);
  // pinned DMA, whole and chunked
  for (int r = 0; r < 2; ++r) {
    auto t = clk::now();
    cudaMemcpyAsync(dev, pin, N, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    printf("pinned DMA 512MB: %.2f ms  %.1f GB/s\n", ms_since(t), N / ms_since(t) / 1e6);
  }
  // memcpy pageable -> pinned with T threads
  for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
    auto t = clk::now();
    std::vector<std::thread> th;
    for (int i = 0; i < T; ++i)
      th.emplace_back([=] { size_t p = N / T; memcpy(pin + i * p, src + i * p, p); });
    for (auto& x : th) x.join();
    printf("memcpy %2d threads: %.2f ms  %.1f GB/s\n", T, ms_since(t), N / ms_since(t) / 1e6);
  }
  // direct pageable DMA
  {
    auto t = clk::now();
    cudaMemcpyAsync(dev, src, N, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    printf("pageable DMA: %.2f ms  %.1f GB/s\n", ms_since(t), N / ms_since(t) / 1e6);
  }
  // register + DMA + unregister
  for (int r = 0; r < 2; ++r) {
    auto t = clk::now();
    cudaError_t e = cudaHostRegister(src, N, cudaHostRegisterDefault);
    double treg = ms_since(t);
    cudaMemcpyAsync(dev, src, N, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    double tdma = ms_since(t) - treg;
    cudaHostUnregister(src);
    printf("register %.2f ms + DMA %.2f ms + unregister -> total %.2f ms (%s)\n", treg, tdma, ms_since(t),
           cudaGetErrorString(e));
  }
  printf("hw threads: %u\n", std::thread::hardware_concurrency());
  return 0;
}
