// Host side of the batched small-matrix kernels (perm_batch_*).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "batch.cuh"
#include "engine.cuh"
#include "walk_launch.cuh"

namespace permb200 {

using batch_fn = cudaError_t (*)(const void*, void*, int64_t, cudaStream_t);

template <typename T>
static cudaError_t prep_smem(const void* kern, size_t smem) {
  if (smem > 48 * 1024)
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

template <typename T, int N>
static cudaError_t launch_bglynn(const void* a, void* out, int64_t B, cudaStream_t s) {
  constexpr int E = N * N;
  constexpr int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const size_t smem = (size_t)kBatchThreads * STRIDE * sizeof(T);
  auto k = batch_glynn_kernel<T, N>;
  cudaError_t e = prep_smem<T>((const void*)k, smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (B + kBatchThreads - 1) / kBatchThreads;
  k<<<(unsigned)grid, kBatchThreads, smem, s>>>(static_cast<const T*>(a), static_cast<T*>(out), B);
  return cudaGetLastError();
}

template <typename T, int M, int N>
static cudaError_t launch_bryser(const void* a, void* out, int64_t B, cudaStream_t s) {
  constexpr int E = M * N;
  constexpr int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const size_t smem = (size_t)kBatchThreads * STRIDE * sizeof(T);
  auto k = batch_ryser_kernel<T, M, N>;
  cudaError_t e = prep_smem<T>((const void*)k, smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (B + kBatchThreads - 1) / kBatchThreads;
  k<<<(unsigned)grid, kBatchThreads, smem, s>>>(static_cast<const T*>(a), static_cast<T*>(out), B);
  return cudaGetLastError();
}

template <typename T, int... Ns>
static batch_fn pick_glynn(int n, std::integer_sequence<int, Ns...>) {
  batch_fn f = nullptr;
  ((n == Ns + 2 ? (f = &launch_bglynn<T, Ns + 2>, 0) : 0), ...);
  return f;
}

// Ryser pairs (M, N), 1 <= M < N <= 12, enumerated (1-based) as
// IDX = (N-1)(N-2)/2 + M
template <typename T, int IDX>
struct RyserPair {
  static constexpr int n_of() {
    int n = 2;
    while (n * (n - 1) / 2 < IDX) ++n;
    return n;
  }
  static constexpr int N = n_of();
  static constexpr int M = IDX - (N - 1) * (N - 2) / 2;
};
template <typename T, int... Is>
static batch_fn pick_ryser(int m, int n, std::integer_sequence<int, Is...>) {
  batch_fn f = nullptr;
  ((m == RyserPair<T, Is + 1>::M && n == RyserPair<T, Is + 1>::N
        ? (f = &launch_bryser<T, RyserPair<T, Is + 1>::M, RyserPair<T, Is + 1>::N>, 0)
        : 0),
   ...);
  return f;
}

template <typename T>
static cudaError_t launch_generic(const void* a, void* out, int64_t B, int m, int n, int alg, cudaStream_t s) {
  const int E = m * n;
  const int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const size_t smem = (size_t)kBatchThreads * STRIDE * sizeof(T);
  auto k = batch_generic_kernel<T>;
  cudaError_t e = prep_smem<T>((const void*)k, smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (B + kBatchThreads - 1) / kBatchThreads;
  k<<<(unsigned)grid, kBatchThreads, smem, s>>>(static_cast<const T*>(a), static_cast<T*>(out), B, m, n, alg);
  return cudaGetLastError();
}

template <typename T, int M, int N>
static cudaError_t launch_bcombdp(const void* a, void* out, int64_t B, cudaStream_t s) {
  constexpr int E = M * N;
  constexpr int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const size_t smem = (size_t)kBatchThreads * STRIDE * sizeof(T);
  auto k = batch_combdp_kernel<T, M, N>;
  cudaError_t e = prep_smem<T>((const void*)k, smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (B + kBatchThreads - 1) / kBatchThreads;
  k<<<(unsigned)grid, kBatchThreads, smem, s>>>(static_cast<const T*>(a), static_cast<T*>(out), B);
  return cudaGetLastError();
}
// (M, N) with 1 <= M <= 4, M <= N <= 12: IDX = (M-1)*12 + (N-1), N >= M
template <typename T, int... Is>
static batch_fn pick_combdp(int m, int n, std::integer_sequence<int, Is...>) {
  batch_fn f = nullptr;
  ((m == Is / 12 + 1 && n == Is % 12 + 1 && Is % 12 + 1 >= Is / 12 + 1
        ? (f = &launch_bcombdp<T, Is / 12 + 1, (Is % 12 + 1 >= Is / 12 + 1 ? Is % 12 + 1 : Is / 12 + 1)>, 0)
        : 0),
   ...);
  return f;
}

using batch_m_fn = cudaError_t (*)(const void*, void*, int64_t, int, cudaStream_t);
template <typename T, int N>
static cudaError_t launch_bglynn_warp(const void* a, void* out, int64_t B, int m, cudaStream_t s) {
  const int64_t grid = (B + kBatchWarpMats - 1) / kBatchWarpMats;
  batch_glynn_warp_kernel<T, N><<<(unsigned)grid, 32 * kBatchWarpMats, 0, s>>>(static_cast<const T*>(a),
                                                                               static_cast<T*>(out), B, m);
  return cudaGetLastError();
}
template <typename T, int... Ns>
static batch_m_fn pick_glynn_warp(int n, std::integer_sequence<int, Ns...>) {
  batch_m_fn f = nullptr;
  ((n == Ns + 9 ? (f = &launch_bglynn_warp<T, Ns + 9>, 0) : 0), ...);
  return f;
}

// Kernel choice for one (device-resident) batch.  The batch-only formulas run
// on the bulk-pipelined kernels when the shape and base address allow (else
// the classic kernel of the same family: Laplace -> Glynn, partition ->
// memoized combinatoric).  Thread-per-matrix needs enough matrices to fill
// the GPU; below that a warp per matrix (n >= 9).
static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Glynn batches of n = 17..30 (square, or rectangular on the ones-padded,
// 2^s-scaled matrix): every matrix's Gray walk split into
// segments over the grid (walk_multi_kernel), partials combined per matrix
// in segment order inside the launch.
static int launch_walk_multi_batch(bool cplx, int64_t B, int m, int n, const void* dA, void* dOut,
                                   cudaStream_t stream) {
  walk_multi_fn fn = walk_multi_lookup(cplx, n);
  walk_multi_bps_fn bfn = walk_multi_bps_lookup(cplx, n);
  if (!fn || !bfn) {
    set_error("no batched walk kernel for this n");
    return PERM_BAD_SHAPE;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  static int bps_cache[2][kWalkMultiMaxN + 1] = {};  // benign race: idempotent
  int& bps = bps_cache[cplx ? 1 : 0][n];
  if (!bps) bps = bfn();
  // at most 2^20 matrices per launch: bounded scratch (partials + counters)
  // however large the device-resident batch
  constexpr int64_t kMaxPerLaunch = 1 << 20;
  const int esz = cplx ? 16 : 8;
  cudaError_t e = cudaSuccess;
  for (int64_t b0 = 0; b0 < B && e == cudaSuccess; b0 += kMaxPerLaunch) {
    const int64_t nb = std::min<int64_t>(kMaxPerLaunch, B - b0);
    const WalkMultiPlan pl = plan_walk_multi(n, nb, nsm, bps);
    const size_t part_bytes = (size_t)nb * pl.segs * kPartialStride * sizeof(double);
    const size_t done_bytes = ((size_t)nb * sizeof(unsigned int) + 255) & ~(size_t)255;
    void* scratch = nullptr;
    e = cudaMallocAsync(&scratch, part_bytes + done_bytes, stream);
    if (e != cudaSuccess) break;
    unsigned int* done = static_cast<unsigned int*>(scratch);
    double* partials = reinterpret_cast<double*>(static_cast<char*>(scratch) + done_bytes);
    e = cudaMemsetAsync(done, 0, (size_t)nb * sizeof(unsigned int), stream);
    if (e == cudaSuccess)
      e = fn(static_cast<const char*>(dA) + (size_t)b0 * m * n * esz, static_cast<char*>(dOut) + (size_t)b0 * esz,
             nb, m, partials, done, pl, stream);
    const cudaError_t ef = cudaFreeAsync(scratch, stream);
    if (e == cudaSuccess) e = ef;
  }
  return e == cudaSuccess ? PERM_OK : cuda_fail(e, "batched walk launch");
}

static int launch_batch(int alg, bool cplx, int64_t B, int m, int n, const void* dA, void* dOut,
                        cudaStream_t stream) {
  if (alg == PERM_ALG_GLYNN && n >= kWalkMultiMinN) return launch_walk_multi_batch(cplx, B, m, n, dA, dOut, stream);
  if (alg == PERM_ALG_BATCH_PARTITION && n > 16) return launch_partition_wide(cplx, B, m, n, dA, dOut, stream);
  if (alg == PERM_ALG_BATCH_LAPLACE || alg == PERM_ALG_BATCH_PARTITION) {
    const int st = launch_bulk_batch(alg, cplx, B, m, n, dA, dOut, stream);
    if (st >= 0) return st;
    alg = (alg == PERM_ALG_BATCH_LAPLACE) ? PERM_ALG_GLYNN
          : (m <= 4)                      ? PERM_ALG_COMBINATORIC  // memoized DP
                                          : PERM_ALG_RYSER;        // subset-skipping
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // large batches: warp per matrix from n = 12 (n = 9..11 thread per matrix is faster; n = 13..16 has no
  // thread-per-matrix template; measured with tools/batch_glynn_large.py)
  static const int warp_min_n = env_int("PERM_BATCH_WARP_MIN_N", 12);
  batch_fn fn = nullptr;
  // warp per matrix: squares as above; rectangles n = 9..16 always (ones-
  // padded, pre-scaled per matrix in the kernel; the runtime-n generic
  // kernel is the only alternative)
  if (alg == PERM_ALG_GLYNN && n >= 9 && n <= 16 && (m < n || B < (int64_t)nsm * 512 || n >= warp_min_n)) {
    batch_m_fn wf = cplx ? pick_glynn_warp<cd>(n, std::make_integer_sequence<int, 8>{})
                         : pick_glynn_warp<double>(n, std::make_integer_sequence<int, 8>{});
    const cudaError_t e = wf(dA, dOut, B, m, stream);
    return e == cudaSuccess ? PERM_OK : cuda_fail(e, "batch kernel launch");
  }
  if (!fn && alg == PERM_ALG_GLYNN && m == n && n >= 2 && n <= 12)
    fn = cplx ? pick_glynn<cd>(n, std::make_integer_sequence<int, 11>{})
              : pick_glynn<double>(n, std::make_integer_sequence<int, 11>{});
  if (!fn && alg == PERM_ALG_COMBINATORIC && m <= 4 && n <= 12)
    fn = cplx ? pick_combdp<cd>(m, n, std::make_integer_sequence<int, 48>{})
              : pick_combdp<double>(m, n, std::make_integer_sequence<int, 48>{});
  if (!fn && alg == PERM_ALG_RYSER && m < n && n <= 12)
    fn = cplx ? pick_ryser<cd>(m, n, std::make_integer_sequence<int, 66>{})
              : pick_ryser<double>(m, n, std::make_integer_sequence<int, 66>{});
  cudaError_t e;
  if (fn) e = fn(dA, dOut, B, stream);
  else e = cplx ? launch_generic<cd>(dA, dOut, B, m, n, alg, stream)
                : launch_generic<double>(dA, dOut, B, m, n, alg, stream);
  return e == cudaSuccess ? PERM_OK : cuda_fail(e, "batch kernel launch");
}

// Two-slot pinned staging for host batches (per host thread, per device).
struct BatchPipe {
  int device = -1;
  void *hin[2] = {nullptr, nullptr}, *hout[2] = {nullptr, nullptr};
  void *din[2] = {nullptr, nullptr}, *dout[2] = {nullptr, nullptr};
  size_t in_cap = 0, out_cap = 0;
  cudaStream_t stream[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int64_t pending[2] = {0, 0}, pending_first[2] = {0, 0};
  int ensure(size_t in_b, size_t out_b) {
    if (!stream[0]) {
      for (int i = 0; i < 2; ++i) {
        PERM_CUDA_TRY(cudaStreamCreateWithFlags(&stream[i], cudaStreamNonBlocking));
        PERM_CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        PERM_CUDA_TRY(cudaEventRecord(done[i], stream[i]));
      }
    }
    if (in_b > in_cap || out_b > out_cap) {
      for (int i = 0; i < 2; ++i) {
        PERM_CUDA_TRY(cudaEventSynchronize(done[i]));
        if (hin[i]) cudaFreeHost(hin[i]);
        if (hout[i]) cudaFreeHost(hout[i]);
        if (din[i]) cudaFree(din[i]);
        if (dout[i]) cudaFree(dout[i]);
        PERM_CUDA_TRY(cudaMallocHost(&hin[i], in_b));
        PERM_CUDA_TRY(cudaMallocHost(&hout[i], out_b));
        PERM_CUDA_TRY(cudaMalloc(&din[i], in_b));
        PERM_CUDA_TRY(cudaMalloc(&dout[i], out_b));
      }
      in_cap = in_b;
      out_cap = out_b;
    }
    return PERM_OK;
  }
};
static thread_local BatchPipe g_pipe[16];
static BatchPipe& batch_pipe() {
  int dev = 0;
  cudaGetDevice(&dev);
  return g_pipe[dev & 15];
}

// Host memcpy split over persistent threads (pageable -> pinned staging).
// Spawning threads per chunk cost ~0.1 ms per chunk; the pool is created on
// first use and lives for the process.  One copy at a time (call_mu).
class CopyPool {
 public:
  void copy(void* dst, const void* src, size_t bytes, int nparts) {
    std::lock_guard<std::mutex> call(call_mu_);
    std::unique_lock<std::mutex> lk(mu_);
    while ((int)nthreads_ < nparts) {
      const int id = (int)nthreads_++;
      std::thread([this, id] { work(id); }).detach();
    }
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    nparts_ = nparts;
    remaining_ = (int)nthreads_;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [this] { return remaining_ == 0; });
  }

 private:
  void work(int id) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      char* d = dst_;
      const char* s = src_;
      const size_t b = bytes_;
      const int np = nparts_;
      lk.unlock();
      if (id < np) {
        const size_t part = ((b + np - 1) / np + 4095) & ~(size_t)4095;
        const size_t off = (size_t)id * part;
        if (off < b) std::memcpy(d + off, s + off, std::min(part, b - off));
      }
      lk.lock();
      if (--remaining_ == 0) done_.notify_all();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  size_t nthreads_ = 0;
  uint64_t gen_ = 0;
  int remaining_ = 0, nparts_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};


static void par_memcpy(void* dst, const void* src, size_t bytes) {
  static CopyPool* pool = new CopyPool();  // detached workers: never destroyed
  const int nt = std::max(1, std::min(32, env_int("PERM_COPY_THREADS", 8)));
  if (bytes < (4u << 20) || nt == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  pool->copy(dst, src, bytes, nt);
}

int batch_select(int m, int n) {
  // cheapest exact per-matrix work: the 4+4 Laplace kernel for 8x8 (1134
  // flops against Glynn's 2048; complex 8x8 falls back to Glynn), Glynn for
  // other squares, the partition formula for m <= 4 (C2b: 290 flops) and for
  // m = 5, 6 with n >= m + 2 (5x10: ~830 flops against ~8300 for the
  // subset-skipping Ryser), that Ryser else
  if (m == 8 && n == 8) return PERM_ALG_BATCH_LAPLACE;
  if (m == n) return PERM_ALG_GLYNN;
  if (m <= 4 || (m <= 6 && n >= m + 2)) return PERM_ALG_BATCH_PARTITION;
  // wider m >= 7 (or m = n - 1) rectangles: Glynn on the ones-padded,
  // pre-scaled matrix -- warp per matrix for n = 9..16 (1e4 x 12x16: 0.74 ms
  // against 31 ms for the subset-skipping Ryser), batched walks above
  if (n >= 9) return PERM_ALG_GLYNN;
  return PERM_ALG_RYSER;
}

// ---------------------------------------------------------------------------
// Zero-copy path for one small matrix from host memory (the batch-of-one
// calls of walk_single).  The matrix is copied into mapped pinned memory, the
// batch kernel reads it over the bus and writes the result back into mapped
// memory, a one-thread kernel then publishes a sequence number, and the host
// spins on it -- one memcpy and two launches instead of H2D + launch + D2H +
// event sync (22 -> ~10 us per call for a 6x6 matrix).
__global__ void tiny_flag_kernel(volatile unsigned int* flag, unsigned int seq) {
  __threadfence_system();
  *flag = seq;
  __threadfence_system();
}

struct TinyBuf {
  int device = -1;
  char* host = nullptr;  // [in 16 KB][out 64 B][flag]
  char* dev = nullptr;   // device alias of host
  cudaStream_t stream = nullptr;
  unsigned int seq = 0;
  static constexpr size_t kIn = 256 * 1024, kOut = 32 * 1024;
  int ensure() {
    int d = 0;
    cudaGetDevice(&d);
    if (host && device == d) return PERM_OK;
    if (host) return PERM_BAD_ARG;  // one buffer per thread: first device only
    PERM_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&host), kIn + kOut + 64, cudaHostAllocMapped));
    PERM_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
    PERM_CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    device = d;
    *reinterpret_cast<volatile unsigned int*>(host + kIn + kOut) = 0;
    return PERM_OK;
  }
};
static thread_local TinyBuf g_tiny;

static bool tiny_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PERM_TINY_ZEROCOPY");
    return !(e && e[0] == '0');
  }();
  return on;
}

// launch the batch kernel on the mapped buffers, publish a sequence number,
// spin until it lands (blocking wait after 2 ms, which also reports errors)
static int tiny_run(TinyBuf& tb, int alg, bool cplx, int64_t B, int m, int n) {
  int st = launch_batch(alg, cplx, B, m, n, tb.dev, tb.dev + TinyBuf::kIn, tb.stream);
  if (st != PERM_OK) return st;
  const unsigned int seq = ++tb.seq;
  volatile unsigned int* hflag = reinterpret_cast<volatile unsigned int*>(tb.host + TinyBuf::kIn + TinyBuf::kOut);
  tiny_flag_kernel<<<1, 1, 0, tb.stream>>>(
      reinterpret_cast<volatile unsigned int*>(tb.dev + TinyBuf::kIn + TinyBuf::kOut), seq);
  PERM_CUDA_TRY(cudaGetLastError());
  const auto t0 = std::chrono::steady_clock::now();
  while (*hflag != seq) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) {
      PERM_CUDA_TRY(cudaStreamSynchronize(tb.stream));
      break;
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return PERM_OK;
}

// A whole small host batch through the mapped buffers (C1: 64 x 12x12).
static int tiny_batch_host(int alg, bool cplx, int64_t B, int m, int n, const double* a, double* out) {
  const size_t esz = cplx ? 16 : 8;
  const size_t in_b = (size_t)B * m * n * esz, out_b = (size_t)B * esz;
  if (!tiny_enabled() || in_b > TinyBuf::kIn || out_b > TinyBuf::kOut) return -1;
  TinyBuf& tb = g_tiny;
  if (tb.ensure() != PERM_OK) return -1;
  std::memcpy(tb.host, a, in_b);
  const int st = tiny_run(tb, alg, cplx, B, m, n);
  if (st != PERM_OK) return st;
  std::memcpy(out, tb.host + TinyBuf::kIn, out_b);
  return PERM_OK;
}

// -1: not taken (caller uses the staged path)
int tiny_permanent(int alg, bool cplx, int m, int n, const double* a, double* out) {
  const size_t esz = cplx ? 16 : 8;
  const size_t bytes = (size_t)m * n * esz;
  if (!tiny_enabled() || bytes > TinyBuf::kIn) return -1;
  TinyBuf& tb = g_tiny;
  if (tb.ensure() != PERM_OK) return -1;
  // Rectangular Glynn: the ones-padded square matrix with the real rows
  // pre-scaled by 2^s (as the walk does, prescale_log2), so the templated
  // square kernel runs; per(A) = per([2^s A; J]) / ((n-m)! 2^(s m)).
  const bool pad = (alg == PERM_ALG_GLYNN && m < n && n <= 12);
  double unscale = 1.0;
  int unscale_exp = 0;
  if (pad) {
    if ((size_t)n * n * esz > TinyBuf::kIn) return -1;
    HostMat A;
    A.m = m;
    A.n = n;
    A.cplx = cplx;
    A.d.assign(a, a + (size_t)m * n * (cplx ? 2 : 1));
    const int sl = prescale_log2(A);
    const double k = std::ldexp(1.0, sl);
    double* h = reinterpret_cast<double*>(tb.host);
    const int w = cplx ? 2 : 1;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int c = 0; c < w; ++c)
          h[((size_t)i * n + j) * w + c] = (i < m) ? a[((size_t)i * n + j) * w + c] * k : (c == 0 ? 1.0 : 0.0);
    double f = 1.0;
    for (int i = 2; i <= n - m; ++i) f *= (double)i;
    unscale = 1.0 / f;
    unscale_exp = -sl * m;  // applied with ldexp on the value (the factor alone can underflow)
  } else {
    std::memcpy(tb.host, a, bytes);
  }
  const int st = tiny_run(tb, alg, cplx, 1, pad ? n : m, n);
  if (st != PERM_OK) return st;
  std::memcpy(out, tb.host + TinyBuf::kIn, esz);
  if (pad) {
    out[0] = std::ldexp(out[0] * unscale, unscale_exp);
    if (cplx) out[1] = std::ldexp(out[1] * unscale, unscale_exp);
  }
  return PERM_OK;
}

int batch_permanent(int alg, bool cplx, int64_t B, int m, int n, const double* a, double* out, int dev_ptr,
                    void* stream_) {
  clear_error();
  if (B < 0 || m < 1 || n < 1 || m > n) {
    set_error(m > n ? "need m <= n; transpose first" : "bad batch shape");
    return PERM_BAD_SHAPE;
  }
  if (alg < 0) {
    alg = batch_select(m, n);
    // the complex partition formula stops at m = 5 (register file)
    if (alg == PERM_ALG_BATCH_PARTITION && cplx && m > 5) alg = (n >= 9) ? PERM_ALG_GLYNN : PERM_ALG_RYSER;
  }
  if (n > 16 && !(alg == PERM_ALG_GLYNN && n <= kWalkMultiMaxN) &&
      !(alg == PERM_ALG_BATCH_PARTITION && n <= 62 && m <= (cplx ? 5 : 6))) {
    set_error("batched kernels handle n <= 16 (Glynn: n <= 30; the partition formula, m <= 6: n <= 62); "
              "use the single-permanent entry points");
    return PERM_BAD_SHAPE;
  }
  if (alg > PERM_ALG_BATCH_LAPLACE) {
    set_error("unknown batch algorithm");
    return PERM_BAD_SHAPE;
  }
  if (alg == PERM_ALG_BATCH_LAPLACE && !(m == 8 && n == 8)) {
    set_error("the Laplace batch formula is 8x8 only");
    return PERM_BAD_SHAPE;
  }
  if (alg == PERM_ALG_BATCH_PARTITION && m > 6) {
    set_error("the partition batch formula needs m <= 6");
    return PERM_BAD_SHAPE;
  }
  if (alg == PERM_ALG_BATCH_LAPLACE && cplx) alg = PERM_ALG_GLYNN;
  if (alg == PERM_ALG_COMBINATORIC) {
    // src/algorithms.py:80-84 budget is per matrix; P(16, 16) would be absurd
    uint64_t perms = 1;
    for (int i = 0; i < m; ++i) perms *= (uint64_t)(n - i);
    if (perms > 2000000000ull) {
      set_error("combinatoric step budget exceeded");
      return PERM_BUDGET;
    }
  }
  if (B == 0) return PERM_OK;
  cudaStream_t stream = pick_stream(stream_);
  const size_t esz = cplx ? 16 : 8;
  const size_t mat_bytes = (size_t)m * n * esz;
  if (dev_ptr) return launch_batch(alg, cplx, B, m, n, a, out, stream);
  if (stream_ == nullptr) {  // small host batches: zero-copy round trip
    const int tst = tiny_batch_host(alg, cplx, B, m, n, a, out);
    if (tst >= 0) return tst;
  }
  // Host arrays: chunked pipeline through two pinned staging slots on two
  // engine streams, so the host copy of chunk c+1, the H2D DMA of chunk c and
  // the kernels overlap (the input is read from pageable numpy memory).
  Scratch* sc = scratch();
  if (!sc) return cuda_fail(cudaErrorNoDevice, "scratch");
  const size_t chunk_bytes = (size_t)std::max(1, env_int("PERM_BATCH_CHUNK_MB", 32)) << 20;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(chunk_bytes / mat_bytes));
  chunk = std::min<int64_t>(chunk, B);
  const size_t in_chunk = (size_t)chunk * mat_bytes, out_chunk = (size_t)chunk * esz;
  BatchPipe& bp = batch_pipe();
  int st = bp.ensure(in_chunk, out_chunk);
  if (st) return st;
  // Page-locked input (cudaHostAlloc / cudaHostRegister, e.g. a pinned torch
  // tensor): the DMA reads the caller's buffer directly, no staging copy.
  bool pinned_in = false;
  {
    // both ends of the array must be page-locked (a cudaHostRegister range
    // may cover only part of it; such input takes the staged route)
    const char* ends[2] = {reinterpret_cast<const char*>(a),
                           reinterpret_cast<const char*>(a) + (size_t)B * mat_bytes - 1};
    pinned_in = true;
    for (const char* p : ends) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();  // an unknown pointer is pageable memory
        pinned_in = false;
      } else if (at.type != cudaMemoryTypeHost) {
        pinned_in = false;
      }
    }
  }
  // Results parked in a slot belong to the call that parked them: drop any
  // left behind by an earlier call that returned early, and drop ours on
  // every early return below, so no later call copies stale results into
  // its own (possibly shorter) output.
  struct SlotReset {
    BatchPipe& bp;
    void drop() {
      for (int slot = 0; slot < 2; ++slot) {
        cudaEventSynchronize(bp.done[slot]);
        bp.pending[slot] = 0;
      }
    }
    ~SlotReset() { drop(); }
  } slot_reset{bp};
  slot_reset.drop();
  for (int64_t c0 = 0, it = 0; c0 < B; c0 += chunk, ++it) {
    const int slot = (int)(it & 1);
    const int64_t cnt = std::min<int64_t>(chunk, B - c0);
    // slot reuse: wait for its previous chunk, then hand its results back
    PERM_CUDA_TRY(cudaEventSynchronize(bp.done[slot]));
    if (bp.pending[slot] > 0) {
      std::memcpy(reinterpret_cast<char*>(out) + (size_t)bp.pending_first[slot] * esz, bp.hout[slot],
                  (size_t)bp.pending[slot] * esz);
      bp.pending[slot] = 0;
    }
    const char* src = reinterpret_cast<const char*>(a) + (size_t)c0 * mat_bytes;
    if (!pinned_in) {
      par_memcpy(bp.hin[slot], src, (size_t)cnt * mat_bytes);
      src = static_cast<const char*>(bp.hin[slot]);
    }
    PERM_CUDA_TRY(cudaMemcpyAsync(bp.din[slot], src, (size_t)cnt * mat_bytes, cudaMemcpyHostToDevice,
                                  bp.stream[slot]));
    st = launch_batch(alg, cplx, cnt, m, n, bp.din[slot], bp.dout[slot], bp.stream[slot]);
    if (st) return st;
    PERM_CUDA_TRY(cudaMemcpyAsync(bp.hout[slot], bp.dout[slot], (size_t)cnt * esz, cudaMemcpyDeviceToHost,
                                  bp.stream[slot]));
    PERM_CUDA_TRY(cudaEventRecord(bp.done[slot], bp.stream[slot]));
    bp.pending[slot] = cnt;
    bp.pending_first[slot] = c0;
  }
  for (int slot = 0; slot < 2; ++slot) {
    PERM_CUDA_TRY(cudaEventSynchronize(bp.done[slot]));
    if (bp.pending[slot] > 0) {
      std::memcpy(reinterpret_cast<char*>(out) + (size_t)bp.pending_first[slot] * esz, bp.hout[slot],
                  (size_t)bp.pending[slot] * esz);
      bp.pending[slot] = 0;
    }
  }
  return PERM_OK;
}

}  // namespace permb200
