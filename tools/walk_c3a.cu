// C3a-sized complex walk (P = 24, B = 23: 2^23 steps) vs chunk length and
// launch shape: the small-walk end of the walk kernel (latency-bound).
#include <cstdio>
#include <random>
#include <string>
#include <vector>
#include "../paper_2510_03421_b200/csrc/walk_launch.cuh"
using namespace permb200;
template <typename T, int P>
void run(int B, int r) {
  const int w = sizeof(T) / 8;
  std::vector<double> h((size_t)(P + B * P) * w);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(-0.05, 0.05);
  for (auto& x : h) x = U(g);
  double *d, *parts;
  unsigned int* dn;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&parts, kMaxPartials * kPartialStride * 8);
  cudaMalloc(&dn, 4);
  cudaMemset(dn, 0, 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  WalkJob job{};
  job.P = P; job.B = B; job.v0 = d; job.U = d + P * w; job.k_begin = 0; job.k_end = 1ull << B;
  job.partials = parts; job.final_out = parts + (size_t)(kMaxPartials - 1) * kPartialStride; job.done = dn;
  job.force_log2L = r;
  WalkPlan plan;
  for (int i = 0; i < 3; ++i) launch_walk<T, P, false>(job, &plan, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch_walk<T, P, false>(job, &plan, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double ops = (double)(1ull << B) * (sizeof(T) == 8 ? 2 * P : 6 * P - 2);
  printf("%s P=%d B=%d r=%d(plan %d) grid=%d threads=%d: %.4f ms %.2f Tops %s\n", sizeof(T) == 8 ? "f64" : "c128", P, B, r,
         plan.log2L, plan.grid, kWalkThreads, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); cudaFree(parts); cudaFree(dn);
}
// modes: (none) C3a chunk sweep; "floor" small-walk floor; "lsweep" chunk
// length sweep at P = 22, 26, 28 (the cost model's check)
int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  if (mode == "floor") {
    for (int b : {13, 15, 17, 19, 21, 23}) run<double, 24>(b, 0);
    for (int b : {13, 17, 19, 21, 23}) run<cd, 24>(b, 0);
    for (int b : {19, 21, 23, 25}) run<double, 36>(b, 0);
  } else if (mode == "lsweep") {
    for (int r : {0, 4, 5, 6, 7, 8, 9, 10}) run<double, 26>(25, r);
    for (int r : {0, 5, 6, 7, 8, 9, 10}) run<double, 28>(27, r);
    for (int r : {0, 4, 5, 6, 7, 8}) run<double, 22>(21, r);
  } else {
    for (int r : {0, 3, 4, 5, 6, 7}) run<cd, 24>(23, r);
    for (int r : {0, 4, 5, 6}) run<double, 24>(23, r);
    for (int r : {0, 4, 5, 6}) run<double, 26>(25, r);
  }
  return 0;
}
