// Per-P sweep of the walk kernel (fixed Gray-range size), for choosing the
// product-chain count per state length.  Prints "T P chains Tops".
#include <cstdio>
#include <random>
#include <utility>
#include <vector>
#include "../paper_2510_03421_b200/csrc/walk_launch.cuh"
using namespace permb200;
template <typename T, int P>
void one(int B) {
  const int w = sizeof(T) / 8;
  std::vector<double> h((size_t)(P + B * P) * w);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(-0.05, 0.05);
  for (auto& x : h) x = U(g);
  double *d, *parts;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&parts, kMaxPartials * kPartialStride * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  WalkJob job{};
  job.P = P; job.B = B; job.v0 = d; job.U = d + P * w; job.k_begin = 0; job.k_end = 1ull << B; job.partials = parts; job.final_out = parts + (size_t)(kMaxPartials - 1) * kPartialStride; { static unsigned int* dn = nullptr; if (!dn) { cudaMalloc(&dn, 4); cudaMemset(dn, 0, 4); } job.done = dn; }
  WalkPlan plan;
  launch_walk<T, P, false>(job, &plan, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 4; ++i) launch_walk<T, P, false>(job, &plan, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 4;
  const double ops = (double)(1ull << B) * (sizeof(T) == 8 ? 2 * P : 6 * P - 2);
  printf("%s %d %d %d %.3f\n", sizeof(T) == 8 ? "f64" : "c128", P, walk_chains<T, P>(), (int)walk_r0<T, P>(),
         ops / (ms * 1e-3) / 1e12);
  cudaFree(d); cudaFree(parts);
}
template <int... Ps> void runf(std::integer_sequence<int, Ps...>) { (one<double, Ps + 12>(std::min(Ps + 11, 29)), ...); }
template <int... Ps> void runc(std::integer_sequence<int, Ps...>) { (one<cd, Ps + 12>(std::min(Ps + 11, 26)), ...); }
template <int... Ps> void runc2(std::integer_sequence<int, Ps...>) { (one<cd, Ps + 20>(std::min(Ps + 19, 26)), ...); }
int main() {
#ifdef CSWEEP_C128_ONLY
  runc2(std::make_integer_sequence<int, 13>{});  // P = 20..32
  return 0;
#endif
  runf(std::make_integer_sequence<int, 41>{});  // P = 12..52
#ifndef CSWEEP_F64_ONLY
  runc(std::make_integer_sequence<int, 25>{});  // P = 12..36
#endif
  return 0;
}
