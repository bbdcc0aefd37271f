// Chunk-length sweep for the Gray-walk kernel (P = 30, 34, 36 real).
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_2510_03421_b200/csrc/walk_launch.cuh"
using namespace permb200;
template <int P>
void sweep(int B) {
  std::vector<double> h((size_t)(P + B * P));
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(-0.05, 0.05);
  for (auto& x : h) x = U(g);
  double *d, *parts;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&parts, kMaxPartials * kPartialStride * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  for (int r = 0; r <= 0; ++r) {
    WalkJob job{};
    job.P = P; job.B = B; job.v0 = d; job.U = d + P; job.k_begin = 0; job.k_end = 1ull << B;
    job.partials = parts; job.final_out = parts + (size_t)(kMaxPartials - 1) * kPartialStride; { static unsigned int* dn = nullptr; if (!dn) { cudaMalloc(&dn, 4); cudaMemset(dn, 0, 4); } job.done = dn; } job.force_log2L = r;
    WalkPlan plan;
    launch_walk<double, P, false>(job, &plan, 0);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = B >= 34 ? 2 : 8;
    for (int i = 0; i < reps; ++i) launch_walk<double, P, false>(job, &plan, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    printf("P=%d B=%d r=%d(plan %d) grid=%d: %.3f ms %.2f Tops\n", P, B, r, plan.log2L, plan.grid, ms,
           (double)(1ull << B) * 2 * P / (ms * 1e-3) / 1e12);
  }
  cudaFree(d); cudaFree(parts);
}
int main() { sweep<26>(25); sweep<28>(27); sweep<30>(29); sweep<32>(31); sweep<34>(33); sweep<36>(35); return 0; }
