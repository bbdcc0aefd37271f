// Host side of the bulk-pipelined batch kernels (batch_bulk.cuh): the
// partition-formula kernel for m <= 6 and the 8x8 row-recursion kernel,
// picked by the batch dispatch (perm_batch_select) for device-resident
// batches that meet the 1-D bulk-copy rules (16-byte aligned base, matrix
// size a multiple of 16 bytes).
#include <algorithm>
#include <utility>

#include "batch_bulk.cuh"
#include "engine.cuh"

namespace permb200 {

namespace {

using bulk_fn = cudaError_t (*)(const void*, void*, int64_t, cudaStream_t);

int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 15;
}
int sm_count() {
  static int nsm[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = nsm[dev & 15];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Tile shape from the matrix size: <= ~40 KB per stage, two stages; as many
// blocks per SM as ~200 KB of shared memory holds, at most 8 (C2b: 4x10
// f64, 128 threads, 2 blocks per SM, 6.0 TB/s).
template <typename T, int M, int N>
struct PartCfg {
  static constexpr int kBytes = M * N * (int)sizeof(T);
  static constexpr int kTPB = kBytes <= 320 ? 128 : (kBytes <= 640 ? 64 : 32);
  static constexpr int kStages = 2;
  static constexpr int kSmem = kStages * kTPB * kBytes;
  static constexpr int kPerSM = (200 * 1024 / kSmem < 1) ? 1 : (200 * 1024 / kSmem > 8 ? 8 : 200 * 1024 / kSmem);
};

template <typename T, int M, int N>
cudaError_t launch_partition(const void* a, void* out, int64_t B, cudaStream_t s) {
  using Cfg = PartCfg<T, M, N>;
  auto k = batch_bulk_kernel<T, M, N, Cfg::kTPB, Cfg::kStages, PartitionOp<T, M, N>>;
  const size_t smem = (size_t)Cfg::kStages * Cfg::kTPB * Cfg::kBytes;
  static bool attr[16] = {false};  // per instantiation and device; idempotent, so racing first calls are harmless
  if (!attr[cur_device()]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[cur_device()] = true;
  }
  const int64_t ntiles = (B + Cfg::kTPB - 1) / Cfg::kTPB;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)Cfg::kPerSM * sm_count());
  k<<<grid, Cfg::kTPB, smem, s>>>(static_cast<const T*>(a), static_cast<T*>(out), B);
  return cudaGetLastError();
}

// 8x8: the row-by-row subset recursion with its middle level parked in TMEM
// (RowDp8Tm), one 8-warp CTA per SM, each warp a single-stage 16 KB tile ring
// (128 KB of shared memory, so one CTA per SM and its 512 TMEM columns).
// C2a 1e6 x 8x8: 0.089 ms, 5.8 TB/s (round 1: 0.115 ms with the shared-memory
// 4+4 Laplace kernel; tools/bulk_bench.cu).
constexpr int kDp8Warps = 8;
cudaError_t launch_laplace8(const void* a, void* out, int64_t B, cudaStream_t s) {
  auto k = perm8_tmem_kernel<kDp8Warps, RowDp8Tm<8>>;
  const size_t smem = (size_t)kDp8Warps * 32 * 64 * sizeof(double);
  static bool attr[16] = {false};
  if (!attr[cur_device()]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[cur_device()] = true;
  }
  const int64_t ntiles = (B + 31) / 32;
  const int grid = (int)std::min<int64_t>((ntiles + kDp8Warps - 1) / kDp8Warps, (int64_t)sm_count());
  k<<<grid, 32 * kDp8Warps, smem, s>>>(static_cast<const double*>(a), static_cast<double*>(out), B);
  return cudaGetLastError();
}

// (M, N), 1 <= M <= 6, M <= N <= 16: IDX = (M-1)*16 + (N-1); f64 needs even
// N (16-byte row chunks); complex stops at M = 5 (M = 6: the 64 complex
// subset sums spill)
template <typename T, int I>
bulk_fn part_entry() {
  constexpr int M = I / 16 + 1, N = I % 16 + 1;
  if constexpr (N >= M && (sizeof(T) == 16 ? M <= 5 : N % 2 == 0)) return &launch_partition<T, M, N>;
  else return nullptr;
}
template <typename T, int... Is>
bulk_fn pick_partition(int m, int n, std::integer_sequence<int, Is...>) {
  bulk_fn f = nullptr;
  ((m == Is / 16 + 1 && n == Is % 16 + 1 ? (f = part_entry<T, Is>(), 0) : 0), ...);
  return f;
}

template <typename T, int M>
cudaError_t launch_partition_rt(const void* a, void* out, int64_t B, int n, cudaStream_t s) {
  const int64_t grid = (B + 127) / 128;
  partition_rt_kernel<T, M><<<(unsigned)grid, 128, 0, s>>>(static_cast<const T*>(a), static_cast<T*>(out), B, n);
  return cudaGetLastError();
}
using rt_fn = cudaError_t (*)(const void*, void*, int64_t, int, cudaStream_t);
template <typename T, int... Ms>
rt_fn pick_rt(int m, std::integer_sequence<int, Ms...>) {
  rt_fn f = nullptr;
  ((m == Ms + 1 ? (f = &launch_partition_rt<T, Ms + 1>, 0) : 0), ...);
  return f;
}

}  // namespace

// Partition formula for wide rectangles, 16 < n <= 62 (m <= 6 real, m <= 4
// complex): runtime-n kernel (no bulk staging).
int launch_partition_wide(bool cplx, int64_t B, int m, int n, const void* dA, void* dOut, cudaStream_t stream) {
  rt_fn fn = cplx ? pick_rt<cd>(m, std::make_integer_sequence<int, 5>{})
                  : pick_rt<double>(m, std::make_integer_sequence<int, 6>{});
  if (!fn || n > 62 || m > n) {
    set_error("the partition batch formula covers m <= 6 (complex m <= 5), n <= 62");
    return PERM_BAD_SHAPE;
  }
  const cudaError_t e = fn(dA, dOut, B, n, stream);
  return e == cudaSuccess ? PERM_OK : cuda_fail(e, "partition batch launch");
}

bool bulk_batch_supported(int alg, bool cplx, int m, int n) {
  if (alg == PERM_ALG_BATCH_LAPLACE) return !cplx && m == 8 && n == 8;
  if (alg == PERM_ALG_BATCH_PARTITION)
    return m >= 1 && m <= n && n <= 16 && (cplx ? m <= 5 : (m <= 6 && n % 2 == 0));
  return false;
}

// Returns PERM_OK, a CUDA failure, or -1 when this (alg, shape, pointer)
// has no bulk kernel (the caller then uses the classic kernels).
int launch_bulk_batch(int alg, bool cplx, int64_t B, int m, int n, const void* dA, void* dOut, cudaStream_t stream) {
  if (!bulk_batch_supported(alg, cplx, m, n)) return -1;
  if ((reinterpret_cast<uintptr_t>(dA) & 15) != 0) return -1;  // 1-D bulk copies need 16-byte addresses
  bulk_fn fn = nullptr;
  if (alg == PERM_ALG_BATCH_LAPLACE) {
    fn = &launch_laplace8;
  } else {
    fn = cplx ? pick_partition<cd>(m, n, std::make_integer_sequence<int, 80>{})
              : pick_partition<double>(m, n, std::make_integer_sequence<int, 96>{});
  }
  if (!fn) return -1;
  const cudaError_t e = fn(dA, dOut, B, stream);
  return e == cudaSuccess ? PERM_OK : cuda_fail(e, "bulk batch kernel launch");
}

}  // namespace permb200
