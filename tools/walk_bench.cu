// Variant harness for the Gray-walk kernel: times walk_kernel on the C5 /
// C3a / C3b shapes with random data (compile with different -D knobs).
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2510_03421_b200/csrc/walk_launch.cuh"
using namespace permb200;

template <typename T, int P>
double run(int B, int reps) {
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
  job.P = P; job.B = B; job.v0 = d; job.U = d + P * w; job.mag = 0;
  job.k_begin = 0; job.k_end = 1ull << B; job.partials = parts; job.final_out = parts + (size_t)(kMaxPartials - 1) * kPartialStride; { static unsigned int* dn = nullptr; if (!dn) { cudaMalloc(&dn, 4); cudaMemset(dn, 0, 4); } job.done = dn; }
  WalkPlan plan;
  launch_walk<T, P, false>(job, &plan, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch_walk<T, P, false>(job, &plan, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double ops = (double)(1ull << B) * (sizeof(T) == 8 ? 2 * P : 6 * P - 2);
  printf("  P=%d %s B=%d: %.3f ms  %.3e steps/s  %.2f Tops/s  (grid %d, log2L %d) err=%s\n", P,
         sizeof(T) == 8 ? "f64" : "c128", B, ms, (1ull << B) / (ms * 1e-3), ops / (ms * 1e-3) / 1e12, plan.grid,
         plan.log2L, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); cudaFree(parts);
  return ms;
}
int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == '3') {  // P = 36 only (profiling)
    run<double, 36>(35, 1);
    return 0;
  }
  if (argc > 1) {  // quick functional check
    run<double, 28>(20, 1);
    run<cd, 24>(18, 1);
    return 0;
  }
  run<double, 36>(35, 3);
  run<double, 32>(31, 10);
  run<double, 28>(27, 20);
  run<cd, 24>(23, 50);
  run<cd, 28>(27, 10);
  return 0;
}
