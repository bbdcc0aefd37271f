// Host side of the batched small-matrix kernels (perm_batch_*).
#include <utility>

#include "batch.cuh"
#include "engine.cuh"

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

int batch_select(int m, int n) {
  // thread-per-matrix fast paths: Glynn for squares, subset-skipping Ryser
  // for rectangles (cheapest exact per-matrix work for C2a / C2b)
  return (m == n) ? PERM_ALG_GLYNN : PERM_ALG_RYSER;
}

int batch_permanent(int alg, bool cplx, int64_t B, int m, int n, const double* a, double* out, int dev_ptr,
                    void* stream_) {
  clear_error();
  if (B < 0 || m < 1 || n < 1 || m > n) {
    set_error(m > n ? "need m <= n; transpose first" : "bad batch shape");
    return PERM_BAD_SHAPE;
  }
  if (n > 16) {
    set_error("batched kernels handle n <= 16; use the single-permanent entry points");
    return PERM_BAD_SHAPE;
  }
  if (alg < 0) alg = batch_select(m, n);
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
  const size_t in_bytes = (size_t)B * m * n * esz, out_bytes = (size_t)B * esz;
  const void* dA = a;
  void* dOut = out;
  void* buf = nullptr;
  if (!dev_ptr) {
    PERM_CUDA_TRY(cudaMallocAsync(&buf, in_bytes + out_bytes + 256, stream));
    dA = buf;
    dOut = static_cast<char*>(buf) + ((in_bytes + 255) & ~(size_t)255);
    PERM_CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(dA), a, in_bytes, cudaMemcpyHostToDevice, stream));
  }
  batch_fn fn = nullptr;
  if (alg == PERM_ALG_GLYNN && m == n && n >= 2 && n <= 12)
    fn = cplx ? pick_glynn<cd>(n, std::make_integer_sequence<int, 11>{})
              : pick_glynn<double>(n, std::make_integer_sequence<int, 11>{});
  if (alg == PERM_ALG_RYSER && m < n && n <= 12)
    fn = cplx ? pick_ryser<cd>(m, n, std::make_integer_sequence<int, 66>{})
              : pick_ryser<double>(m, n, std::make_integer_sequence<int, 66>{});
  cudaError_t e;
  if (fn) e = fn(dA, dOut, B, stream);
  else e = cplx ? launch_generic<cd>(dA, dOut, B, m, n, alg, stream)
                : launch_generic<double>(dA, dOut, B, m, n, alg, stream);
  if (e != cudaSuccess) {
    if (buf) cudaFreeAsync(buf, stream);
    return cuda_fail(e, "batch kernel launch");
  }
  if (!dev_ptr) {
    PERM_CUDA_TRY(cudaMemcpyAsync(out, dOut, out_bytes, cudaMemcpyDeviceToHost, stream));
    PERM_CUDA_TRY(cudaFreeAsync(buf, stream));
    PERM_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  return PERM_OK;
}

}  // namespace permb200
