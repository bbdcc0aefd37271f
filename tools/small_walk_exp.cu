// Small single walks (n = 14..26): where the time goes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -ffp-contract=off \
//        -I paper_2510_03421_b200/csrc tools/small_walk_exp.cu -o tools/swx_small      (add -DWALK_TIMELINE
//        for the per-phase %globaltimer stamps of the walk kernel)
//   tools/swx_small                    launch floors, then P = 16..36: setup in device memory + D2H copy
//                                      vs setup as kernel parameters + mapped result flag
//   SKIP_FLOOR=1 tools/swx_small       the walks only;  BIG=1: P = 30..34;  N24=1: chunk-length sweep
//
// Launch floors: an empty kernel back to back (device time per launch) and
// launch -> host-visible round trips (stream sync vs a flag in mapped host
// memory), with 0 / 4 / 8 / 16 / 30 KB of kernel parameters.  Results:
// DESIGN 2.3b, profiles/r2_small_walk_probe.txt.  (Variants measured and
// dropped there: an all-lanes-contiguous work split, per-block partials
// published straight to host memory.)
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "walk_launch.cuh"

using namespace permb200;
using clk = std::chrono::steady_clock;
static unsigned *g_hflag, *g_dflag;
static double *g_hres, *g_dres;

template <int BYTES>
struct Blob {
  double d[BYTES / 8 > 0 ? BYTES / 8 : 1];
};

template <int BYTES>
__global__ void param_kernel(const __grid_constant__ Blob<BYTES> b, double* out, volatile unsigned* flag,
                             unsigned seq) {
  extern __shared__ double sm[];
  constexpr int N = BYTES / 8;
  for (int i = threadIdx.x; i < N; i += blockDim.x) sm[i] = b.d[i];
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = N ? sm[N - 1] : 0.0;
    if (flag) {
      __threadfence_system();
      *flag = seq;
    }
  }
}

static double us_since(clk::time_point t) { return std::chrono::duration<double, std::micro>(clk::now() - t).count(); }

static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

template <int BYTES>
void launch_floor(double* dout, unsigned* hflag, unsigned* dflag, int grid) {
  Blob<BYTES> b;
  for (int i = 0; i < (int)(sizeof(b.d) / 8); ++i) b.d[i] = i;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const size_t smem = BYTES > 0 ? BYTES : 8;
  cudaFuncSetAttribute(param_kernel<BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int i = 0; i < 50; ++i) param_kernel<BYTES><<<grid, 256, smem, s>>>(b, dout, nullptr, 0);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int R = 500;
  cudaEventRecord(e0, s);
  for (int i = 0; i < R; ++i) param_kernel<BYTES><<<grid, 256, smem, s>>>(b, dout, nullptr, 0);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> rt_sync, rt_flag, host_launch;
  for (int i = 0; i < 300; ++i) {
    auto t = clk::now();
    param_kernel<BYTES><<<grid, 256, smem, s>>>(b, dout, nullptr, 0);
    host_launch.push_back(us_since(t));
    cudaStreamSynchronize(s);
    rt_sync.push_back(us_since(t));
  }
  static unsigned seq = 0;
  for (int i = 0; i < 300; ++i) {
    ++seq;
    auto t = clk::now();
    param_kernel<BYTES><<<grid, 256, smem, s>>>(b, dout, dflag, seq);
    while (*(volatile unsigned*)hflag != seq) {
    }
    rt_flag.push_back(us_since(t));
  }
  cudaStreamSynchronize(s);
  printf("params %5d B grid %3d: back-to-back %6.2f us/launch  host launch %5.2f us  round trip sync %6.2f us  "
         "flag %6.2f us\n",
         BYTES, grid, 1e3 * ms / R, median(host_launch), median(rt_sync), median(rt_flag));
  cudaStreamDestroy(s);
}

template <int P>
void walk_exp(double* d_part, double* d_final, unsigned* d_done, double* d_data) {
  const int B = P - 1;
  constexpr int PS = row_stride<double, P>();
  (void)PS;
  // C5 law: U[0,1]/n
  std::vector<double> a((size_t)P * P), buf((size_t)P + (size_t)B * P);
  unsigned long long x = 88172645463325252ull + P;
  for (auto& v : a) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = (double)(x >> 11) * 0x1.0p-53 / P;
  }
  for (int j = 0; j < P; ++j) {
    double c = 0;
    for (int i = 0; i < P; ++i) c += a[(size_t)i * P + j];
    buf[j] = c;
  }
  for (int t = 0; t < B; ++t)
    for (int j = 0; j < P; ++j) buf[P + (size_t)t * P + j] = -2.0 * a[(size_t)(P - 1 - t) * P + j];
  cudaMemcpy(d_data, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  WalkJob job{};
  job.dtype = 0;
  job.P = P;
  job.B = B;
  job.weighted = false;
  job.v0 = d_data;
  job.U = d_data + P;
  job.w = nullptr;
  job.wlen = 0;
  job.mag = 0;
  job.k_begin = 0;
  job.k_end = 1ull << B;
  job.partials = d_part;
  job.final_out = d_final;
  job.done = d_done;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  static unsigned seq = 0;
  // modes: 0 setup in device memory, result by D2H copy + stream sync;
  // 1 setup as kernel parameters, result + flag in mapped host memory
  for (int mode = 0; mode < 2; ++mode) {
    job.inline_host = mode == 1 && walk_inline_ok<double, P, false>() ? buf.data() : nullptr;
    job.flag = nullptr;
    WalkPlan plan;
    for (int i = 0; i < 20; ++i) launch_walk<double, P, false>(job, &plan, s);
    cudaStreamSynchronize(s);
    const int R = P > 30 ? 5 : 200;
    cudaEventRecord(e0, s);
    for (int i = 0; i < R; ++i) launch_walk<double, P, false>(job, &plan, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<double> rt;
    double h[8];
    for (int i = 0; i < (P > 30 ? 3 : 100); ++i) {
      auto t = clk::now();
      if (mode == 0) {
        launch_walk<double, P, false>(job, &plan, s);
        cudaMemcpyAsync(h, d_final, 64, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
      } else {
        job.flag = g_dflag;
        job.final_out = g_dres;
        job.seq = ++seq;
        launch_walk<double, P, false>(job, &plan, s);
        while (*(volatile unsigned*)g_hflag != seq) {
        }
        std::memcpy(h, g_hres, 64);
        job.flag = nullptr;
        job.final_out = d_final;
      }
      rt.push_back(us_since(t));
    }
    const double us = 1e3 * ms / R;
    const double pipe = (double)(1ull << B) * 2 * P / (us * 1e-6) / (148 * 64 * 1.965e9);
    printf("P=%d %-18s grid %4d log2L %2d: back-to-back %9.2f us/launch (pipe %5.1f%%)  call round trip %9.2f us  "
           "value %.15e\n",
           P, mode == 0 ? "global+copy" : (job.inline_host ? "inline+flag" : "global+flag"), plan.grid, plan.log2L,
           us, 100 * pipe, median(rt), h[0] + h[1]);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      exit(1);
    }
  }
#ifdef WALK_TIMELINE
  {
    unsigned long long* d_tl;
    cudaMalloc(&d_tl, 4096 * 8 * 8);
    cudaMemcpyToSymbol(g_walk_tl, &d_tl, sizeof(d_tl));
    job.inline_host = walk_inline_ok<double, P, false>() ? buf.data() : nullptr;
    WalkPlan plan;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(d_tl, 0, 4096 * 64);
      job.seq = ++seq;
      launch_walk<double, P, false>(job, &plan, s);
      cudaStreamSynchronize(s);
    }
    std::vector<unsigned long long> tl((size_t)plan.grid * 8);
    cudaMemcpy(tl.data(), d_tl, tl.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0min = ~0ull, t0max = 0, t4max = 0, t3max = 0;
    double ph[4] = {0, 0, 0, 0};
    for (int b = 0; b < plan.grid; ++b) {
      const unsigned long long* t = &tl[(size_t)b * 8];
      t0min = std::min(t0min, t[0]);
      t0max = std::max(t0max, t[0]);
      t3max = std::max(t3max, t[3]);
      t4max = std::max(t4max, t[4]);
      for (int k = 0; k < 4; ++k) ph[k] += (double)(t[k + 1] - t[k]) / plan.grid;
    }
    printf("P=%d timeline%s (ns, grid %d): block start spread %llu | stage %.0f | seed+walk %.0f | block reduce %.0f | "
           "combine %.0f (avg) | last t3 -> end %llu | span %llu\n",
           P, "", plan.grid, t0max - t0min, ph[0], ph[1], ph[2], ph[3], t4max - t3max,
           t4max - t0min);
    unsigned long long* z = nullptr;
    cudaMemcpyToSymbol(g_walk_tl, &z, sizeof(z));
    cudaFree(d_tl);
    job.inline_host = nullptr;
  }
#endif
  cudaStreamDestroy(s);
}

// N24=1: the n = 24 walk over forced chunk lengths (and whatever WALK_*
// macros this binary was built with)
template <int P>
void chunk_sweep(double* d_part, double* d_final, unsigned* d_done, double* d_data) {
  const int B = P - 1;
  std::vector<double> a((size_t)P * P), buf((size_t)P + (size_t)B * P);
  unsigned long long x = 88172645463325252ull + P;
  for (auto& v : a) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = (double)(x >> 11) * 0x1.0p-53 / P;
  }
  for (int j = 0; j < P; ++j) {
    double c = 0;
    for (int i = 0; i < P; ++i) c += a[(size_t)i * P + j];
    buf[j] = c;
  }
  for (int t = 0; t < B; ++t)
    for (int j = 0; j < P; ++j) buf[P + (size_t)t * P + j] = -2.0 * a[(size_t)(P - 1 - t) * P + j];
  cudaMemcpy(d_data, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  WalkJob job{};
  job.P = P; job.B = B; job.v0 = d_data; job.U = d_data + P; job.k_begin = 0; job.k_end = 1ull << B;
  job.partials = d_part; job.final_out = d_final; job.done = d_done;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r : {0, 4, 5, 6, 7, 8}) {
    job.force_log2L = r;
    WalkPlan plan;
    for (int i = 0; i < 20; ++i) launch_walk<double, P, false>(job, &plan, s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 200; ++i) launch_walk<double, P, false>(job, &plan, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / 200;
    printf("P=%d r0=%d log2L %d%s grid %d: %.2f us (pipe %.1f%%)\n", P, (int)walk_r0<double, P>(), plan.log2L,
           r ? "" : " (model)", plan.grid, us, 100.0 * (double)(1ull << B) * 2 * P / (us * 1e-6) / (148 * 64 * 1.965e9));
  }
}

int main() {
  if (getenv("N24")) {
    double *d_part, *d_final, *d_data;
    unsigned* d_done;
    cudaMalloc(&d_part, (size_t)kMaxPartials * kPartialStride * 8);
    cudaMalloc(&d_final, 64);
    cudaMalloc(&d_data, 1 << 20);
    cudaMalloc(&d_done, 4);
    cudaMemset(d_done, 0, 4);
    chunk_sweep<22>(d_part, d_final, d_done, d_data);
    chunk_sweep<23>(d_part, d_final, d_done, d_data);
    chunk_sweep<24>(d_part, d_final, d_done, d_data);
    chunk_sweep<25>(d_part, d_final, d_done, d_data);
    return 0;
  }
  if (getenv("BIG")) {
    double *d_part, *d_final, *d_data;
    unsigned* d_done;
    cudaMalloc(&d_part, (size_t)kMaxPartials * kPartialStride * 8);
    cudaMalloc(&d_final, 64);
    cudaMalloc(&d_data, 1 << 20);
    cudaMalloc(&d_done, 4);
    cudaMemset(d_done, 0, 4);
    walk_exp<30>(d_part, d_final, d_done, d_data);
    walk_exp<31>(d_part, d_final, d_done, d_data);
    walk_exp<32>(d_part, d_final, d_done, d_data);
    walk_exp<33>(d_part, d_final, d_done, d_data);
    walk_exp<34>(d_part, d_final, d_done, d_data);
    return 0;
  }
  double *d_part, *d_final, *d_data, *d_out;
  unsigned *d_done, *hflag, *dflag;
  cudaMalloc(&d_part, (size_t)kMaxPartials * kPartialStride * 8);
  cudaMalloc(&d_final, 64);
  cudaMalloc(&d_data, 1 << 20);
  cudaMalloc(&d_out, 64);
  cudaMalloc(&d_done, 4);
  cudaMemset(d_done, 0, 4);
  cudaHostAlloc(&hflag, 64, cudaHostAllocMapped);
  *hflag = 0;
  cudaHostGetDevicePointer(&dflag, hflag, 0);
  cudaHostAlloc(&g_hflag, 64, cudaHostAllocMapped);
  *g_hflag = 0;
  cudaHostGetDevicePointer(&g_dflag, g_hflag, 0);
  cudaHostAlloc(&g_hres, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&g_dres, g_hres, 0);
  for (int g : {148}) {
    if (getenv("SKIP_FLOOR")) break;
    launch_floor<0>(d_out, hflag, dflag, g);
    launch_floor<4096>(d_out, hflag, dflag, g);
    launch_floor<8192>(d_out, hflag, dflag, g);
    launch_floor<16384>(d_out, hflag, dflag, g);
    launch_floor<30720>(d_out, hflag, dflag, g);
  }
  walk_exp<16>(d_part, d_final, d_done, d_data);
  walk_exp<18>(d_part, d_final, d_done, d_data);
  walk_exp<20>(d_part, d_final, d_done, d_data);
  walk_exp<22>(d_part, d_final, d_done, d_data);
  walk_exp<24>(d_part, d_final, d_done, d_data);
  walk_exp<26>(d_part, d_final, d_done, d_data);
  walk_exp<28>(d_part, d_final, d_done, d_data);
  walk_exp<32>(d_part, d_final, d_done, d_data);
  walk_exp<36>(d_part, d_final, d_done, d_data);
  return 0;
}
