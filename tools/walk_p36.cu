// Walk-kernel variant harness at the headline state length (P = 36 real,
// Glynn-like unweighted walk, 2^31 steps): compile with -DWALK_CHAINS=K
// -DWALK_CHAINS_FIXED -DWALK_MINB=b -DWALK_THREADS=t to compare product-chain
// counts / register caps.  Prints "chains minb threads grid ms Tops".
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_2510_03421_b200/csrc/walk_launch.cuh"
using namespace permb200;
template <int P>
void run(int B) {
  std::vector<double> h((size_t)(P + B * P));
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
  job.P = P; job.B = B; job.v0 = d; job.U = d + P; job.k_begin = 0; job.k_end = 1ull << B;
  job.partials = parts; job.final_out = parts + (size_t)(kMaxPartials - 1) * kPartialStride; job.done = dn;
  WalkPlan plan;
  launch_walk<double, P, false>(job, &plan, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) launch_walk<double, P, false>(job, &plan, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  double res[8];
  cudaMemcpy(res, job.final_out, 64, cudaMemcpyDeviceToHost);
  printf("P=%d chains=%d minb=%d threads=%d grid=%d log2L=%d: %.3f ms %.3f Tops  sum=%.17g %s\n", P, walk_chains<double, P>(),
         walk_min_blocks<double, P>(), kWalkThreads, plan.grid, plan.log2L, ms,
         (double)(1ull << B) * 2 * P / (ms * 1e-3) / 1e12, res[0] + res[1], cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<36>(31);
  run<32>(30);
  run<28>(28);
  return 0;
}
