// Batched small permanents (north_star item 4): one thread per matrix.
//
// A block of kBatchThreads threads owns kBatchThreads consecutive matrices:
// it copies their contiguous bytes global -> shared with coalesced 16-byte
// loads (the batch is row-major contiguous [B][m][n]), each matrix padded to
// an odd number of 8-byte words so the per-thread row reads that follow are
// bank-conflict free, then every thread walks its own matrix in registers.
// All threads walk the *same* Gray index sequence, so every branch (flip row,
// direction, subset-size skip) is warp-uniform.
//
//   Glynn, square N <= 12 (C2a: 8x8): 2^(N-1) steps of N adds + (N-1) muls,
//     the three most frequent flip rows (3/4... 7/8 of all steps) held in
//     registers as -2*row, the rest read from shared memory.
//   Ryser, rectangular M < N <= 12 (C2b: 4x10): all 2^N column subsets in
//     Gray order with M-entry row sums; the product is formed only when the
//     subset size s <= M (the binomial weight is 0 above, src/algorithms.py:
//     110-115) -- a uniform branch, so C2b costs 1023 * M adds + 385 products.
//   Generic (runtime m <= n <= 16, any algorithm): the same walks with
//     runtime loops, for shapes without a template.
#pragma once
#include "common.cuh"
#include "walk.cuh"

namespace permb200 {

#ifndef BATCH_THREADS
#define BATCH_THREADS 32
#endif
constexpr int kBatchThreads = BATCH_THREADS;

template <typename T>
__device__ __forceinline__ void batch_stage(const T* __restrict__ g, T* s, int64_t first, int64_t count, int E,
                                            int stride) {
  // copy `count` matrices of E elements starting at matrix `first` into smem
  // with per-matrix stride `stride` (elements)
  const int64_t base = first * E;
  const int64_t total = count * E;
  const double* gd = reinterpret_cast<const double*>(g + base);
  constexpr int W = sizeof(T) / 8;  // doubles per element
  const int64_t nd = total * W;
  if ((reinterpret_cast<uintptr_t>(gd) & 15) == 0) {
    const double2* g2 = reinterpret_cast<const double2*>(gd);
    for (int64_t i = threadIdx.x; i < nd / 2; i += blockDim.x) {
      double2 x = g2[i];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t d = 2 * i + h;
        const int64_t e = d / W;
        const int64_t t = e / E, r = e - t * E;
        reinterpret_cast<double*>(s + t * stride + r)[d - e * W] = h ? x.y : x.x;
      }
    }
    if (nd & 1) {
      const int64_t d = nd - 1;
      if (threadIdx.x == 0) {
        const int64_t e = d / W;
        const int64_t t = e / E, r = e - t * E;
        reinterpret_cast<double*>(s + t * stride + r)[d - e * W] = gd[d];
      }
    }
  } else {
    for (int64_t d = threadIdx.x; d < nd; d += blockDim.x) {
      const int64_t e = d / W;
      const int64_t t = e / E, r = e - t * E;
      reinterpret_cast<double*>(s + t * stride + r)[d - e * W] = gd[d];
    }
  }
}

template <typename T, int P>
__device__ __forceinline__ T prod_chain(const T (&v)[P]) {
  if constexpr (P == 1) return v[0];
  T a = v[0], b = v[1];
#pragma unroll
  for (int j = 2; j < P; j += 2) {
    a = Num<T>::mul(a, v[j]);
    if (j + 1 < P) b = Num<T>::mul(b, v[j + 1]);
  }
  return Num<T>::mul(a, b);
}

// ---------------------------------------------------------------- Glynn
template <typename T, int N>
__device__ T batch_glynn_one(const T* __restrict__ A /* smem, row stride N */) {
  T v[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    T s = A[j];
#pragma unroll
    for (int i = 1; i < N; ++i) s = Num<T>::add(s, A[i * N + j]);
    v[j] = s;
  }
  T acc = prod_chain<T, N>(v);
  if constexpr (N <= 3) {
    // 2^(N-1) <= 4 steps: plain walk
    for (int k = 1; k < (1 << (N - 1)); ++k) {
      const int t = __ffs(k) - 1;
      const bool set = ((k ^ (k >> 1)) >> t) & 1;
      const T* row = A + (N - 1 - t) * N;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const T d = Num<T>::add(row[j], row[j]);
        v[j] = set ? Num<T>::sub(v[j], d) : Num<T>::add(v[j], d);
      }
      const T p = prod_chain<T, N>(v);
      acc = (k & 1) ? Num<T>::sub(acc, p) : Num<T>::add(acc, p);
    }
    return acc;
  } else {
    // hot rows in registers: U[t] = -2 * row(N-1-t), t = 0, 1, 2
    T u0[N], u1[N], u2[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      u0[j] = Num<T>::scale(-2.0, A[(N - 1) * N + j]);
      u1[j] = Num<T>::scale(-2.0, A[(N - 2) * N + j]);
      u2[j] = Num<T>::scale(-2.0, A[(N - 3) * N + j]);
    }
    constexpr int NQ = (1 << (N - 1)) / 8;
    for (int q = 0; q < NQ; ++q) {
      if (q) {
        const int l0 = q << 3;
        const int t = __ffs(l0) - 1;  // >= 3
        const double s = (((l0 ^ (l0 >> 1)) >> t) & 1) ? -2.0 : 2.0;
        const T* row = A + (N - 1 - t) * N;
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = Num<T>::fmas(s, row[j], v[j]);
        acc = Num<T>::add(acc, prod_chain<T, N>(v));
      }
#define PB_STEP(U, OP, SGN)                                                   \
  _Pragma("unroll") for (int j = 0; j < N; ++j) v[j] = Num<T>::OP(v[j], U[j]); \
  acc = Num<T>::SGN(acc, prod_chain<T, N>(v));
      PB_STEP(u0, add, sub)   // l = 1
      PB_STEP(u1, add, add)   // l = 2
      PB_STEP(u0, sub, sub)   // l = 3
      if ((q & 1) == 0) {     // l = 4: bit 2 set iff bit 3 of 8q clear
        PB_STEP(u2, add, add)
      } else {
        PB_STEP(u2, sub, add)
      }
      PB_STEP(u0, add, sub)   // l = 5
      PB_STEP(u1, sub, add)   // l = 6
      PB_STEP(u0, sub, sub)   // l = 7
#undef PB_STEP
    }
    return acc;
  }
}

template <typename T, int N>
__global__ void __launch_bounds__(kBatchThreads) batch_glynn_kernel(const T* __restrict__ a, T* __restrict__ out,
                                                                    int64_t nbatch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);
  constexpr int E = N * N;
  constexpr int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const int64_t first = (int64_t)blockIdx.x * kBatchThreads;
  const int64_t count = (nbatch - first < kBatchThreads) ? nbatch - first : kBatchThreads;
  batch_stage<T>(a, s, first, count, E, STRIDE);
  __syncthreads();
  if (threadIdx.x < count) {
    const T acc = batch_glynn_one<T, N>(s + threadIdx.x * STRIDE);
    out[first + threadIdx.x] = Num<T>::scale(1.0 / (double)(1 << (N - 1)), acc);
  }
}

// -------------------------------------------------------- Glynn, warp/matrix
// For batches too small to fill the device with one thread per matrix (C1:
// 64 x 12x12), a warp walks one matrix: lane l owns the Gray chunk
// [l*L, (l+1)*L), L = 2^(N-1)/32, and runs the same fused 8-step walk as
// walk_kernel on the matrix's -2*rows staged in shared memory (warp-uniform
// reads: broadcasts).  Needs N >= 9 (L >= 8).
constexpr int kBatchWarpMats = 8;  // matrices (warps) per block

template <typename T, int N>
__global__ void __launch_bounds__(32 * kBatchWarpMats) batch_glynn_warp_kernel(const T* __restrict__ a,
                                                                              T* __restrict__ out, int64_t nbatch,
                                                                              int m) {
  // m < N: rectangular Glynn on [2^s A; J] (ones rows below the m real rows,
  // s = round(-log2 RMS of the nonzero entries) per matrix, as prescale_log2)
  constexpr int PS = row_stride<T, N>();
  constexpr int SLOT = (N - 1) * PS + PS;  // U rows + column sums
  __shared__ __align__(16) T smem[kBatchWarpMats * SLOT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mat = (int64_t)blockIdx.x * kBatchWarpMats + warp;
  if (mat >= nbatch) return;  // whole warp exits together
  T* sU = smem + warp * SLOT;
  T* sV0 = sU + (N - 1) * PS;
  const T* A = a + mat * m * N;
  int sl = 0;
  if (m < N) {
    double ss = 0.0;
    int nz = 0;
    for (int e = lane; e < m * N; e += 32) {
      const double q = Num<T>::re(A[e]) * Num<T>::re(A[e]) + Num<T>::im(A[e]) * Num<T>::im(A[e]);
      if (q != 0.0) {
        ss += q;
        ++nz;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, off);
      nz += __shfl_xor_sync(0xffffffffu, nz, off);
    }
    if (nz > 0 && ss > 0.0) {
      const double e = -0.5 * log2(ss / nz);
      if (isfinite(e)) sl = (int)rint(e);
    }
  }
  const double k = ldexp(1.0, sl);
  for (int e = lane; e < N * N; e += 32) {
    const int i = e / N, j = e - i * N;
    if (i >= 1)  // U[t] = -2 row(N-1-t)
      sU[(N - 1 - i) * PS + j] = (i < m) ? Num<T>::scale(-2.0 * k, A[e]) : Num<T>::scale(-2.0, Num<T>::one());
  }
  for (int j = lane; j < N; j += 32) {
    T s = Num<T>::zero();
    for (int i = 0; i < m; ++i) s = Num<T>::add(s, A[i * N + j]);
    sV0[j] = Num<T>::add(Num<T>::scale(k, s), Num<T>::scale((double)(N - m), Num<T>::one()));
  }
  __syncwarp();
  constexpr int LOG2L = N - 1 - 5;
  const uint64_t k0 = (uint64_t)lane << LOG2L;
  const uint64_t g0 = k0 ^ (k0 >> 1);
  T v[N];
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = sV0[j];
  for (int t = LOG2L - 1; t < N - 1; ++t)
    if ((g0 >> t) & 1) row_add<T, N>(v, sU + t * PS);
  double mag = 0.0;
  T acc = walk_chunk_fused<T, N, false, false>(v, sU, nullptr, k0, 1ull << (LOG2L - 3), 0, mag);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if constexpr (sizeof(T) == 8) {
      acc = acc + __shfl_down_sync(0xffffffffu, acc, off);
    } else {
      acc.x += __shfl_down_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_down_sync(0xffffffffu, acc.y, off);
    }
  }
  if (lane == 0) {
    double f = (double)(1 << (N - 1));
    for (int i = 2; i <= N - m; ++i) f *= (double)i;
    const T r = Num<T>::scale(1.0 / f, acc);
    if constexpr (sizeof(T) == 8) out[mat] = ldexp(r, -sl * m);
    else out[mat] = cd_make(ldexp(r.x, -sl * m), ldexp(r.y, -sl * m));
  }
}

// ---------------------------------------------------------------- Ryser
template <typename T, int M, int N>
__device__ T batch_ryser_one(const T* __restrict__ A /* smem, row stride N */, const double* __restrict__ w) {
  T v[M];
#pragma unroll
  for (int i = 0; i < M; ++i) v[i] = Num<T>::zero();
  T acc = Num<T>::zero();
  int pc = 0;
  if constexpr (N < 3) {
    for (int k = 1; k < (1 << N); ++k) {
      const int t = __ffs(k) - 1;
      const bool set = ((k ^ (k >> 1)) >> t) & 1;
#pragma unroll
      for (int i = 0; i < M; ++i) v[i] = set ? Num<T>::add(v[i], A[i * N + t]) : Num<T>::sub(v[i], A[i * N + t]);
      pc += set ? 1 : -1;
      if (pc <= M) acc = Num<T>::add(acc, Num<T>::scale(w[pc], prod_chain<T, M>(v)));
    }
    return acc;
  } else {
    // columns 0, 1, 2 (7 of every 8 flips) in registers; Gray schedule
    // unrolled by 8 as in batch_glynn_one; subsets larger than M skipped
    // (their weight is 0) -- pc is the same for every thread: uniform branch
    T c0[M], c1[M], c2[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      c0[i] = A[i * N + 0];
      c1[i] = A[i * N + 1];
      c2[i] = A[i * N + 2];
    }
#define RB_TERM()                                                                   \
  if (pc <= M) acc = Num<T>::add(acc, Num<T>::scale(w[pc], prod_chain<T, M>(v)));
#define RB_STEP(C, OP, D)                                                           \
  _Pragma("unroll") for (int i = 0; i < M; ++i) v[i] = Num<T>::OP(v[i], C[i]);    \
  pc += D;                                                                          \
  RB_TERM()
    constexpr int NQ = (1 << N) / 8;
    for (int q = 0; q < NQ; ++q) {
      if (q) {
        const int l0 = q << 3;
        const int t = __ffs(l0) - 1;  // >= 3
        const bool set = ((l0 ^ (l0 >> 1)) >> t) & 1;
#pragma unroll
        for (int i = 0; i < M; ++i)
          v[i] = set ? Num<T>::add(v[i], A[i * N + t]) : Num<T>::sub(v[i], A[i * N + t]);
        pc += set ? 1 : -1;
        RB_TERM()
      }
      RB_STEP(c0, add, 1)   // l = 1
      RB_STEP(c1, add, 1)   // l = 2
      RB_STEP(c0, sub, -1)  // l = 3
      if ((q & 1) == 0) {   // l = 4
        RB_STEP(c2, add, 1)
      } else {
        RB_STEP(c2, sub, -1)
      }
      RB_STEP(c0, add, 1)   // l = 5
      RB_STEP(c1, sub, -1)  // l = 6
      RB_STEP(c0, sub, -1)  // l = 7
    }
#undef RB_STEP
#undef RB_TERM
    return acc;
  }
}

template <typename T, int M, int N>
__global__ void __launch_bounds__(kBatchThreads) batch_ryser_kernel(const T* __restrict__ a, T* __restrict__ out,
                                                                    int64_t nbatch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double w[N + 1];
  T* s = reinterpret_cast<T*>(smem_raw);
  constexpr int E = M * N;
  constexpr int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  if (threadIdx.x <= N) {
    // (-1)^(m-s) C(n-s, m-s), zero above m (src/algorithms.py:110-115)
    const int sz = threadIdx.x;
    double c = 0.0;
    if (sz >= 1 && sz <= M) {
      c = 1.0;
      for (int i = 1; i <= M - sz; ++i) c = c * (double)(N - M + i) / (double)i;
      if ((M - sz) & 1) c = -c;
    }
    w[sz] = c;
  }
  const int64_t first = (int64_t)blockIdx.x * kBatchThreads;
  const int64_t count = (nbatch - first < kBatchThreads) ? nbatch - first : kBatchThreads;
  batch_stage<T>(a, s, first, count, E, STRIDE);
  __syncthreads();
  if (threadIdx.x < count) {
    T acc = batch_ryser_one<T, M, N>(s + threadIdx.x * STRIDE, w);
    if (M == N && (N & 1) == 0) {
      // square: weights (-1)^(n-s) already carry the sign
    }
    out[first + threadIdx.x] = acc;
  }
}

// ------------------------------------------------ combinatoric, memoized DP
// The combinatoric sum over m-permutations (src/_kernels.py:28-56) with its
// prefix products memoized over column *sets*:
//   f_1({j}) = a_0j,  f_k(S) = sum_{j in S} a_{k-1,j} f_{k-1}(S \ {j}),
//   per = sum_{|T| = m-1} f_{m-1}(T) * (R_{m-1} - sum_{j in T} a_{m-1,j}),
// R_i the row sum.  For very rectangular shapes (m <= 4) this costs
// sum_k k C(n,k) flops -- 4x10 (C2b): 90 + 120 x 7 = 930 FP64 ops against
// 1023 x 4 + 385 x 5 for the subset-skipping Ryser -- with every index
// compile-time (pairs f_2 in registers).  Exact algebra; sums of products.
template <typename T, int M, int N>
__device__ T batch_combdp_one(const T* __restrict__ A /* smem, row stride N */) {
  T acc = Num<T>::zero();
  if constexpr (M == 1) {
#pragma unroll
    for (int j = 0; j < N; ++j) acc = Num<T>::add(acc, A[j]);
    return acc;
  } else {
    // row sum of the last row
    T R = Num<T>::zero();
#pragma unroll
    for (int j = 0; j < N; ++j) R = Num<T>::add(R, A[(M - 1) * N + j]);
    if constexpr (M == 2) {
      // per = sum_i a0i (R1 - a1i)
#pragma unroll
      for (int i = 0; i < N; ++i) acc = Num<T>::add(acc, Num<T>::mul(A[i], Num<T>::sub(R, A[N + i])));
      return acc;
    } else if constexpr (M == 3) {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
          const T f2 = Num<T>::add(Num<T>::mul(A[N + i], A[j]), Num<T>::mul(A[N + j], A[i]));
          const T g = Num<T>::sub(Num<T>::sub(R, A[2 * N + i]), A[2 * N + j]);
          acc = Num<T>::add(acc, Num<T>::mul(f2, g));
        }
      return acc;
    } else {
      static_assert(M == 4, "memoized DP kernel covers m <= 4");
      constexpr int NP = N * (N - 1) / 2;
      T f2[NP];
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j)
          f2[i * N - i * (i + 1) / 2 + (j - i - 1)] =
              Num<T>::add(Num<T>::mul(A[N + i], A[j]), Num<T>::mul(A[N + j], A[i]));
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j)
#pragma unroll
          for (int k = j + 1; k < N; ++k) {
            const T fij = f2[i * N - i * (i + 1) / 2 + (j - i - 1)];
            const T fik = f2[i * N - i * (i + 1) / 2 + (k - i - 1)];
            const T fjk = f2[j * N - j * (j + 1) / 2 + (k - j - 1)];
            const T f3 = Num<T>::add(Num<T>::add(Num<T>::mul(A[2 * N + i], fjk), Num<T>::mul(A[2 * N + j], fik)),
                                     Num<T>::mul(A[2 * N + k], fij));
            const T g = Num<T>::sub(Num<T>::sub(Num<T>::sub(R, A[3 * N + i]), A[3 * N + j]), A[3 * N + k]);
            acc = Num<T>::add(acc, Num<T>::mul(f3, g));
          }
      return acc;
    }
  }
}

template <typename T, int M, int N>
__global__ void __launch_bounds__(kBatchThreads) batch_combdp_kernel(const T* __restrict__ a, T* __restrict__ out,
                                                                     int64_t nbatch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);
  constexpr int E = M * N;
  constexpr int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const int64_t first = (int64_t)blockIdx.x * kBatchThreads;
  const int64_t count = (nbatch - first < kBatchThreads) ? nbatch - first : kBatchThreads;
  batch_stage<T>(a, s, first, count, E, STRIDE);
  __syncthreads();
  if (threadIdx.x < count) out[first + threadIdx.x] = batch_combdp_one<T, M, N>(s + threadIdx.x * STRIDE);
}

// ---------------------------------------------------------------- generic
// Runtime m <= n <= 16; alg 0 combinatoric (DFS over m-permutations),
// 1 Ryser (all-subsets with weights), 2 Glynn (ones-padded, pre-scaled rows).
template <typename T>
__global__ void __launch_bounds__(kBatchThreads) batch_generic_kernel(const T* __restrict__ a, T* __restrict__ out,
                                                                      int64_t nbatch, int m, int n, int alg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);
  const int E = m * n;
  const int STRIDE = (sizeof(T) == 8) ? (E | 1) : E + 1;
  const int64_t first = (int64_t)blockIdx.x * kBatchThreads;
  const int64_t count = (nbatch - first < kBatchThreads) ? nbatch - first : kBatchThreads;
  batch_stage<T>(a, s, first, count, E, STRIDE);
  __syncthreads();
  if (threadIdx.x >= count) return;
  const T* A = s + threadIdx.x * STRIDE;
  T result = Num<T>::zero();
  if (alg == 1) {
    double w[17];
    for (int sz = 0; sz <= n; ++sz) {
      double c = 0.0;
      if (sz >= 1 && sz <= m) {
        c = 1.0;
        for (int i = 1; i <= m - sz; ++i) c = c * (double)(n - m + i) / (double)i;
        if ((m - sz) & 1) c = -c;
      }
      w[sz] = c;
    }
    T v[16];
    for (int i = 0; i < m; ++i) v[i] = Num<T>::zero();
    int pc = 0;
    for (int k = 1; k < (1 << n); ++k) {
      const int t = __ffs(k) - 1;
      const bool set = ((k ^ (k >> 1)) >> t) & 1;
      for (int i = 0; i < m; ++i) v[i] = set ? Num<T>::add(v[i], A[i * n + t]) : Num<T>::sub(v[i], A[i * n + t]);
      pc += set ? 1 : -1;
      if (pc <= m) {
        T p = v[0];
        for (int i = 1; i < m; ++i) p = Num<T>::mul(p, v[i]);
        result = Num<T>::add(result, Num<T>::scale(w[pc], p));
      }
    }
  } else if (alg == 2) {
    // pre-scale the real rows by k = 2^round(-log2 RMS)
    // (RMS over the nonzero entries, as prescale_log2 on the host)
    double ss = 0.0;
    int nz = 0;
    for (int e = 0; e < E; ++e) {
      const double x = Num<T>::re(A[e]), y = Num<T>::im(A[e]);
      const double q = x * x + y * y;
      if (q != 0.0) {
        ss += q;
        ++nz;
      }
    }
    int sl = 0;
    if (m < n && nz > 0) sl = (int)rint(-0.5 * log2(ss / (double)nz));
    T v[16];
    for (int j = 0; j < n; ++j) {
      T c = Num<T>::zero();
      for (int i = 0; i < m; ++i) c = Num<T>::add(c, Num<T>::scale(ldexp(1.0, sl), A[i * n + j]));
      v[j] = Num<T>::add(c, Num<T>::scale((double)(n - m), Num<T>::one()));
    }
    T p = v[0];
    for (int j = 1; j < n; ++j) p = Num<T>::mul(p, v[j]);
    result = p;
    for (int k = 1; k < (1 << (n - 1)); ++k) {
      const int t = __ffs(k) - 1;
      const int row = n - 1 - t;
      const bool set = ((k ^ (k >> 1)) >> t) & 1;
      const double sg = set ? -2.0 : 2.0;
      for (int j = 0; j < n; ++j) {
        const T x = (row < m) ? Num<T>::scale(ldexp(1.0, sl), A[row * n + j]) : Num<T>::one();
        v[j] = Num<T>::fmas(sg, x, v[j]);
      }
      p = v[0];
      for (int j = 1; j < n; ++j) p = Num<T>::mul(p, v[j]);
      result = (k & 1) ? Num<T>::sub(result, p) : Num<T>::add(result, p);
    }
    double f = 1.0;
    for (int i = 2; i <= n - m; ++i) f *= (double)i;
    result = Num<T>::scale(ldexp(1.0, -(n - 1) - m * sl) / f, result);
  } else {
    // DFS over m-permutations with prefix products (src/_kernels.py:28-56)
    int ch[16];
    bool used[16];
    T prod[17];
    for (int j = 0; j < n; ++j) used[j] = false;
    for (int i = 0; i < m; ++i) ch[i] = -1;
    prod[0] = Num<T>::one();
    int d = 0;
    while (d >= 0) {
      int j = ch[d];
      if (j >= 0) used[j] = false;
      ++j;
      while (j < n && used[j]) ++j;
      if (j >= n) { ch[d] = -1; --d; continue; }
      ch[d] = j;
      const T p = Num<T>::mul(prod[d], A[d * n + j]);
      if (d == m - 1) {
        result = Num<T>::add(result, p);
      } else if (Num<T>::re(p) != 0.0 || Num<T>::im(p) != 0.0) {
        used[j] = true;
        prod[d + 1] = p;
        ++d;
      }
    }
  }
  out[first + threadIdx.x] = result;
}

}  // namespace permb200
